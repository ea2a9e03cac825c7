# compute-sanitizer racecheck + synccheck on a small mixed run; out dir = $1
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 200 python tools/san_mixed.py > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?" >> $OUT/racecheck.log; tail -4 $OUT/racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 200 python tools/san_mixed.py > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?" >> $OUT/synccheck.log; tail -4 $OUT/synccheck.log
