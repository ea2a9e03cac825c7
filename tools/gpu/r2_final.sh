# round-2 evidence: smoke, full GPU suite, bench line, microbenchmarks,
# compute-sanitizer; out dir = $1
OUT=gpurun_out/${1:-r2final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-200 $OUT/bench.json
for m in mb_sync mb_round mb_sort mb_barmix mb_clock; do timeout 120 tools/microbench/$m > $OUT/$m.txt 2>&1; done
timeout 200 python tools/s2_timeline.py --ops 16 > $OUT/s2_timeline.txt 2>&1
bash tools/gpu/san.sh ${1:-r2final}/san
