# round-end check of the committed state: smoke, full GPU suite, bench
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread 2>&1 | tail -8 > gpurun_out/final/pytest_gpu_all.log
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
cat gpurun_out/final/smoke.log gpurun_out/final/pytest_gpu_all.log gpurun_out/final/bench.json
