# seed-bound width experiment: C2 bench and C3 sweep per IVFTQ_SEED_P
for p in 1 2 4; do
  export IVFTQ_SEED_P=$p
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_seed$p.log 2>&1
  tail -1 gpurun_out/bench_seed$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('P=$p', d['value'], d['roofline']['kernel_ms'], d['recall_at_10'])"
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && IVFTQ_SEED_P=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seed_bound -c 3 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep seed | awk -F'","' '{print $(NF)}'
