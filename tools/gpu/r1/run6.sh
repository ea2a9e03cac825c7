# r03 evidence: bench line, reference arm, launch list, ncu --set full of the
# deleteMin and insert launches, mixed-workload and K-sweep probes
mkdir -p gpurun_out/r03
timeout 600 python bench.py > gpurun_out/r03/bench.json 2> gpurun_out/r03/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r03/bench_ref.json 2> gpurun_out/r03/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r03/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03/b_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel -c 2 -o gpurun_out/r03/full_phases -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/r03/full.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/r03/probe_profile.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/r03/probe_ksweep.log 2>&1
timeout 400 python tools/probe_mixed.py --ref > gpurun_out/r03/probe_mixed.log 2>&1
cat gpurun_out/r03/bench.json gpurun_out/r03/probe_profile.log gpurun_out/r03/probe_ksweep.log gpurun_out/r03/probe_mixed.log
