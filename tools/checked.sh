#!/bin/bash
# The checked build (-DPM_FLOW_CHECKED=1: device-side bounds/invariant asserts in the
# scheduled engine) over tools/sanitize_cases.py at several sizes and the flow tests.
make variant VNAME=checked VFLAGS="-DPM_FLOW_CHECKED=1" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
PM_LIB=libparmerge_b200_checked.so python tools/sanitize_cases.py 4096 65536 262144 1048576 3000000 > gpurun_out/r2_checked_cases.log 2>&1
echo "cases rc=$?" > gpurun_out/r2_checked_summary.txt
PM_LIB=libparmerge_b200_checked.so python -m pytest tests/test_flow_gpu.py tests/test_adversarial_gpu.py -q -x > gpurun_out/r2_checked_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_checked_summary.txt
tail -2 gpurun_out/r2_checked_pytest.log >> gpurun_out/r2_checked_summary.txt
