mkdir -p gpurun_out/ds
timeout 120 python tools/probe_phase.py --log2n 20 --k 1024 > gpurun_out/ds/q20.log 2>&1; echo "rc=$?" >> gpurun_out/ds/q20.log
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/ds/q26p.log 2>&1; echo "rc=$?" >> gpurun_out/ds/q26p.log
timeout 120 python tools/probe_phase.py --log2n 26 --k 256 512 1024 2048 > gpurun_out/ds/q26.log 2>&1; echo "rc=$?" >> gpurun_out/ds/q26.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -5 > gpurun_out/ds/pytest.log
cat gpurun_out/ds/q20.log gpurun_out/ds/q26p.log gpurun_out/ds/q26.log gpurun_out/ds/pytest.log
