# quick iteration: GPU tests, trace stats, bench line, ncu instruction count of the headline scan
timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python scripts/trace_scan.py 1000000 64 > gpurun_out/trace.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'], d['recall_at_10'], [(s['nprobe'], round(s['qps'])) for s in d['sweep']])"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:scan_tc_kernel -s 9 -c 1 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '"(gpu__time|smsp__inst|sm__pipe|smsp__issue)' | awk -F'","' '{print $(NF-2), $NF}'
