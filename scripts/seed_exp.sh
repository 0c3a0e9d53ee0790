timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in 0 1; do
  if [ $v = 1 ]; then export IVFTQ_NO_SEED=1; fi
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_seed$v.log 2>&1
  tail -1 gpurun_out/bench_seed$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noseed=$v', d['value'], d['roofline']['kernel_ms'], d['recall_at_10'])"
  timeout 900 python scripts/scale_run.py --config c3 --parity-queries 100 --parity-rows 1000 > gpurun_out/c3_seed$v.log 2>&1
  grep -E '"nprobe": (16|32|64|128), "(qps|queries)' gpurun_out/c3_seed$v.log | cut -c1-220
done
