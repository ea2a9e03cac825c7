mkdir -p gpurun_out/r03
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel --launch-skip 1 -c 1 -o gpurun_out/r03/full_delete -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/r03/full_delete.log 2>&1
tail -2 gpurun_out/r03/full_delete.log
