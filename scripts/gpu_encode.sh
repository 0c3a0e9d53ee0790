# tensor-core encoder: every GPU parity test, then device encode rate at C2/C3 shapes against the f64 tail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for a in "1000000 128 1024" "1000000 96 4096" "500000 200 4096"; do
  timeout 200 python scripts/encode_bench.py $a 2>&1 | tail -1
  IVFTQ_ENCODE_F64=1 timeout 200 python scripts/encode_bench.py $a 2>&1 | tail -1
done
