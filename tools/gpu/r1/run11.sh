mkdir -p gpurun_out/ds
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --profile > gpurun_out/ds/p26b.log 2>&1; echo "rc=$?" >> gpurun_out/ds/p26b.log
cat gpurun_out/ds/p26b.log
