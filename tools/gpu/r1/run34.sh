mkdir -p gpurun_out/r09
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r09/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r09/b_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel --launch-skip 1 -c 1 -o gpurun_out/r09/full_delete -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/r09/full.log 2>&1
tail -2 gpurun_out/r09/full.log; ls -la gpurun_out/r09
