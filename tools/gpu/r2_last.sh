# round-2 last evidence run of the committed tree: smoke, GPU suite, bench
# (ours + reference), serving stress, recorded-history stress; out dir = $1
OUT=gpurun_out/${1:-r2last}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-200 $OUT/bench.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-200 $OUT/bench_ref.json
timeout 1500 python tools/stress_serving.py --runs 300 --seed 7 > $OUT/stress_serving.log 2>&1; tail -2 $OUT/stress_serving.log
timeout 1800 python tools/stress_recorded.py 3 > $OUT/stress_recorded.log 2>&1; tail -3 $OUT/stress_recorded.log
