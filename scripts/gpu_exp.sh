# role-bound experiments at C3 shape (scan kernel time per library variant) + the trace
for v in libivftq_b200.so libivftq_b200_exp_nodec.so libivftq_b200_exp_noepi.so libivftq_b200_exp_nomma.so libivftq_b200_exp_nodec_noepi.so; do
  IVFTQ_LIB=paper_2605_17415_b200/lib/$v timeout 300 python scripts/scan_exp.py ${1:-10000000} ${2:-32} ${3:-96} ${4:-4096} 2>&1 | tail -1
done
python scripts/trace_scan.py 10000000 32 96 4096 > gpurun_out/trace_c3.log 2>&1; python scripts/trace_stats.py gpurun_out/trace.txt
