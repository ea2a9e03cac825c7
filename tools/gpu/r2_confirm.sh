# round-2 confirmation of the committed tree: smoke, full GPU suite, bench
# line, K sweep and mixed probes, ncu launch list; out dir = $1
OUT=gpurun_out/${1:-r2confirm}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-200 $OUT/bench.json
timeout 600 python tools/probe_phase.py --k 256 512 1024 2048 > $OUT/probe_ksweep.log 2>&1; cat $OUT/probe_ksweep.log | cut -c1-120
timeout 300 python tools/probe_phase.py --variant td > $OUT/probe_td.log 2>&1; tail -1 $OUT/probe_td.log | cut -c1-120
timeout 300 python tools/probe_mixed.py --variants bu,td --reps 2 > $OUT/probe_mixed.log 2>&1; cat $OUT/probe_mixed.log | cut -c1-140
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.json 2>&1; head -6 $OUT/launches.json
