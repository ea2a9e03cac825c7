mkdir -p gpurun_out/ds
timeout 900 python tools/stress_serving.py --runs 80 --seed 1 > gpurun_out/ds/stress1.log 2>&1; echo "rc=$?" >> gpurun_out/ds/stress1.log
tail -5 gpurun_out/ds/stress1.log; grep -c FAIL gpurun_out/ds/stress1.log
