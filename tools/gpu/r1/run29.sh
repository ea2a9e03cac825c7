timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['delete_ms'], d['insert_ms'], d['e2e']['value'])"
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_serving.py -q --timeout 300 --timeout-method thread 2>&1 | tail -1
