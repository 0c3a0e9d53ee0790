timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/trace_scan.py 1000000 64 > gpurun_out/trace.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'], d['recall_at_10'], [(s['nprobe'], round(s['qps'])) for s in d['sweep']])"
