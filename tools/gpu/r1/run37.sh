mkdir -p gpurun_out/r09
timeout 600 python bench.py > gpurun_out/r09/bench.json 2> gpurun_out/r09/bench.err
cut -c1-200 gpurun_out/r09/bench.json
