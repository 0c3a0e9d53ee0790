# parity, then role-bound experiments (scan kernel time per library variant) + the trace
timeout -k 5 150 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in libivftq_b200.so libivftq_b200_exp_nodec.so libivftq_b200_exp_noepi.so libivftq_b200_exp_nopush.so; do
  IVFTQ_SCAN_VQ=1 IVFTQ_LIB=paper_2605_17415_b200/lib/$v timeout -k 5 120 python scripts/scan_exp.py ${1:-10000000} ${2:-32} ${3:-96} ${4:-4096} 2>&1 | tail -1
done
timeout -k 5 120 python scripts/scan_exp.py 1000000 64 128 1024 2>&1 | tail -1
bash scripts/gpu_vq_trace.sh ${1:-10000000} ${2:-32} ${3:-96} ${4:-4096}
