# delete serving: quick drain check, probe, GPU suite
mkdir -p gpurun_out/ds
timeout 120 python tools/probe_phase.py --log2n 20 --k 1024 > gpurun_out/ds/p20.log 2>&1; echo "p20 rc=$?" >> gpurun_out/ds/p20.log
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/ds/p26.log 2>&1; echo "p26 rc=$?" >> gpurun_out/ds/p26.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -15 > gpurun_out/ds/pytest.log
cat gpurun_out/ds/p20.log gpurun_out/ds/p26.log gpurun_out/ds/pytest.log
