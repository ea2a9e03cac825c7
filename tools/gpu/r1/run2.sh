# correctness first, then the phase probe
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 90 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/probe.log 2>&1
timeout 120 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/probe_ksweep.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/probe.log gpurun_out/probe_ksweep.log
