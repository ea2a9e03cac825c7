# r04 evidence: bench line, reference arm, launch list, ncu capture of the delete launch
mkdir -p gpurun_out/r04
timeout 600 python bench.py > gpurun_out/r04/bench.json 2> gpurun_out/r04/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r04/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r04/b_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel --launch-skip 1 -c 1 -o gpurun_out/r04/full_delete -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/r04/full.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/r04/probe_profile.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/r04/probe_ksweep.log 2>&1
timeout 400 python tools/probe_mixed.py --ref > gpurun_out/r04/probe_mixed.log 2>&1
cat gpurun_out/r04/bench.json gpurun_out/r04/probe_profile.log gpurun_out/r04/probe_ksweep.log gpurun_out/r04/probe_mixed.log
