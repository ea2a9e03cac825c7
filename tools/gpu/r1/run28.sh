mkdir -p gpurun_out/r07
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r07/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread 2>&1 | tail -4 > gpurun_out/r07/pytest_gpu_all.log
timeout 600 python tools/stress_serving.py --runs 400 --seed 5 > gpurun_out/r07/stress_serving.log 2>&1
timeout 600 python bench.py > gpurun_out/r07/bench.json 2> gpurun_out/r07/bench.err
timeout 300 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/r07/probe_ksweep.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 1024 --variant td > gpurun_out/r07/probe_td.log 2>&1
timeout 400 python tools/probe_mixed.py --ref > gpurun_out/r07/probe_mixed.log 2>&1
cat gpurun_out/r07/smoke.log gpurun_out/r07/pytest_gpu_all.log; tail -1 gpurun_out/r07/stress_serving.log; cut -c1-200 gpurun_out/r07/bench.json; cat gpurun_out/r07/probe_ksweep.log gpurun_out/r07/probe_td.log
