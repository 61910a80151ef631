for v in "" _s256 _s512 _s2048 _s4096; do
  PM_LIB=libparmerge_b200$v.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split$v.csv -k regex:k_flow_s python tools/prof_flow.py 29 auto 2 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_flow<" -s 1 -c 1 -o gpurun_out/flow_full python tools/prof_flow.py 29 auto 2 > gpurun_out/flow_full.log 2>&1
