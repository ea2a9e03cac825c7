# round-2 baseline: smoke, bench line, phase profile, GPU tests; out dir = $1
OUT=gpurun_out/${1:-r2full}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-400 $OUT/bench.json
timeout 300 python tools/probe_phase.py --profile > $OUT/probe_profile.log 2>&1; tail -30 $OUT/probe_profile.log
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
