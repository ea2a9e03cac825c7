# three-level server check: serve3 vs serve2 vs none at K=1024, then the phase probe; out dir = $1
# (the library with the server compiled in: make -C paper_1906_06504_b200/csrc SERVE3=1 DEV=1)
export BH_LIB=${BH_LIB:-build_var/libbatchheap_b200_serve3.so}
OUT=gpurun_out/${1:-s3}
mkdir -p $OUT
timeout 240 python tools/check_serve3.py 20 1024 1 > $OUT/check.log 2>&1; echo "rc=$?" >> $OUT/check.log; tail -6 $OUT/check.log
timeout 200 python tools/probe_phase.py --profile > $OUT/probe_profile.log 2>&1; tail -8 $OUT/probe_profile.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
