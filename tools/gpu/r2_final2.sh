# round-2 final evidence of the committed tree (after the same-box A/B
# changes): smoke, GPU suite, bench + reference arm, ncu launch list, full
# captures of the delete and insert launches, stress; out dir = $1
OUT=gpurun_out/${1:-r2final2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-200 $OUT/bench.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-200 $OUT/bench_ref.json
timeout 300 python tools/probe_phase.py --profile > $OUT/probe_profile.log 2>&1; cat $OUT/probe_profile.log | cut -c1-400
timeout 600 python tools/probe_phase.py --k 256 512 1024 2048 > $OUT/probe_ksweep.log 2>&1; cut -c1-120 $OUT/probe_ksweep.log
timeout 300 python tools/probe_phase.py --variant td > $OUT/probe_td.log 2>&1; tail -1 $OUT/probe_td.log | cut -c1-120
timeout 300 python tools/probe_mixed.py --variants bu,td --reps 2 > $OUT/probe_mixed.log 2>&1; cut -c1-140 $OUT/probe_mixed.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.json 2>&1; head -8 $OUT/launches.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:heap_ops_kernel -s 1 -c 1 \
  -o $OUT/del26 python tools/probe_phase.py > $OUT/ncu_full.log 2>&1; tail -1 $OUT/ncu_full.log
python tools/ncu_summary.py full $OUT/del26.ncu-rep bu_k1024_n26_delete > $OUT/ncu_full_delete.json 2>&1; head -12 $OUT/ncu_full_delete.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:heap_ops_kernel -s 0 -c 1 \
  -o $OUT/ins26 python tools/probe_phase.py > $OUT/ncu_full_ins.log 2>&1; tail -1 $OUT/ncu_full_ins.log
python tools/ncu_summary.py full $OUT/ins26.ncu-rep bu_k1024_n26_insert > $OUT/ncu_full_insert.json 2>&1; head -12 $OUT/ncu_full_insert.json
timeout 900 python tools/stress_serving.py --runs 300 --seed 13 > $OUT/stress_serving.log 2>&1; tail -1 $OUT/stress_serving.log
timeout 1800 python tools/stress_recorded.py 3 > $OUT/stress_recorded.log 2>&1; tail -1 $OUT/stress_recorded.log
