# round-2 ncu evidence: launch list of the bench command, one full capture of
# the delete launch at 2^26 / K=1024, reference arm + CPU matrix; out dir = $1
OUT=gpurun_out/${1:-r2ncu}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.json 2>&1; head -20 $OUT/launches.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:heap_ops_kernel -s 1 -c 1 \
  -o $OUT/del26 python tools/probe_phase.py > $OUT/ncu_full.log 2>&1; tail -2 $OUT/ncu_full.log
python tools/ncu_summary.py full $OUT/del26.ncu-rep bu_k1024_n26_delete > $OUT/ncu_full_delete.json 2>&1; head -30 $OUT/ncu_full_delete.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-300 $OUT/bench_ref.json
timeout 900 python tools/ref_matrix.py $OUT/ref_matrix.json > $OUT/ref_matrix.log 2>&1; tail -8 $OUT/ref_matrix.log
