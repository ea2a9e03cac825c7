mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 100000 python tools/diag_phase_check.py ${1:-18} 0x2000 0x0 > /tmp/race.log 2>&1
grep -E "hazard detected|Read Thread|Write Thread|RACECHECK SUMMARY" /tmp/race.log | sed -E 's/block \([0-9]+,0,0\)//; s/Thread \([0-9]+,0,0\)/Thread/; s/__shared__ 0x[0-9a-f]+/smem/; s/\+0x[0-9a-f]+//; s/bh::HeapCta<[^>]*>:://' | sort | uniq -c | sort -rn > gpurun_out/san/race_summary.txt
head -60 gpurun_out/san/race_summary.txt
