# full check: smoke, GPU tests, drain stress (K 256/1024/2048), phase probe; out dir = $1
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for k in 1024 256 2048; do timeout 400 python tools/stress_drain.py 20 4 $k 0x0 0x2000; done > $OUT/stress_drain.log 2>&1; cat $OUT/stress_drain.log
timeout 300 python tools/probe_phase.py --profile > $OUT/probe_profile.log 2>&1; tail -7 $OUT/probe_profile.log
timeout 300 python tools/probe_phase.py > $OUT/probe.log 2>&1; tail -1 $OUT/probe.log
