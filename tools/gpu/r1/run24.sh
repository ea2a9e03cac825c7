# r06 evidence: smoke, full GPU suite, bench line, reference arm, launch list,
# ncu capture of the delete launch, probes
mkdir -p gpurun_out/r06
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r06/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread 2>&1 | tail -4 > gpurun_out/r06/pytest_gpu_all.log
timeout 600 python bench.py > gpurun_out/r06/bench.json 2> gpurun_out/r06/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r06/bench_ref.json 2> gpurun_out/r06/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r06/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r06/b_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:heap_ops_kernel --launch-skip 1 -c 1 -o gpurun_out/r06/full_delete -f python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/r06/full.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/r06/probe_profile.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/r06/probe_ksweep.log 2>&1
timeout 400 python tools/probe_mixed.py --ref > gpurun_out/r06/probe_mixed.log 2>&1
cat gpurun_out/r06/smoke.log gpurun_out/r06/pytest_gpu_all.log gpurun_out/r06/bench.json gpurun_out/r06/probe_ksweep.log
timeout 600 python tools/stress_serving.py --runs 300 --seed 3 > gpurun_out/r06/stress_serving.log 2>&1; tail -1 gpurun_out/r06/stress_serving.log
