mkdir -p gpurun_out/r06
timeout 1200 python tools/apps_bench.py > gpurun_out/r06/apps_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r06/apps_bench.log
cat gpurun_out/r06/apps_bench.log
