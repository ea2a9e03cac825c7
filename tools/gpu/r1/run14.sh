mkdir -p gpurun_out/ds
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel --launch-skip 1 -c 1 -o gpurun_out/ds/full_delete_sv -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/ds/full_delete_sv.log 2>&1
tail -3 gpurun_out/ds/full_delete_sv.log
ls -la gpurun_out/ds/
