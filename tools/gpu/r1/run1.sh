set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/probe.log 2>&1
timeout 300 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/probe_ksweep.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/probe.log gpurun_out/probe_ksweep.log gpurun_out/bench.log
