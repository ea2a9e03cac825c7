# quick hang check with the debug library, then tests and probes
mkdir -p gpurun_out
timeout 40 python tools/diag_wait.py TD 1024 20 2>&1 | grep -v "line   2[34][0-9] tid    0" | tail -20
timeout 40 python tools/diag_wait.py BU 1024 20 2>&1 | grep -v "line   2[34][0-9] tid    0" | tail -20
bash tools/gpu/run2.sh
