#!/bin/bash
# Install the UNMODIFIED reference into baseline/_ref (git-ignored; travels to the GPU
# box with gpurun) plus its tests beside it, for the reference arm and the drop-in test.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refsrc baseline/_ref
cp -r /root/reference/pkg /tmp/refsrc   # (the build writes egg-info into the source tree)
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target baseline/_ref /tmp/refsrc --no-deps -q
cp -r /root/reference/pkg/tests baseline/_ref/ref_tests
echo "installed: $(ls baseline/_ref)"
