# quick GPU check: smoke + phase probe (profile) + bench line; out dir = $1
OUT=gpurun_out/${1:-quick}
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -3 $OUT/smoke.log
timeout 300 python tools/probe_phase.py --profile > $OUT/probe_profile.log 2>&1; tail -8 $OUT/probe_profile.log
timeout 300 python tools/probe_phase.py > $OUT/probe.log 2>&1; tail -3 $OUT/probe.log
