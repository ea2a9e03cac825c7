mkdir -p gpurun_out
timeout 40 python tools/diag_wait.py BU 1024 20 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -4
timeout 300 python tools/probe_mixed.py --reps 1 2>&1 | tail -3
timeout 90 python tools/probe_phase.py --log2n 26 --k 1024 2>&1 | tail -2
