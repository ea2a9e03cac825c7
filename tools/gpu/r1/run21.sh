mkdir -p gpurun_out/ds
timeout 900 python tools/stress_serving.py --runs 600 --seed 2 > gpurun_out/ds/stress2.log 2>&1; echo "rc=$?" >> gpurun_out/ds/stress2.log
tail -3 gpurun_out/ds/stress2.log; grep FAIL gpurun_out/ds/stress2.log | head; true
