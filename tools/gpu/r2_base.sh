mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
cut -c1-300 gpurun_out/r2a/bench.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/probe_phase.py --profile > gpurun_out/r2a/probe_profile.log 2>&1; tail -30 gpurun_out/r2a/probe_profile.log
