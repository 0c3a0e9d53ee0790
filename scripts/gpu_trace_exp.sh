for v in trace trace_nodec_noepi trace_nopush; do
  echo "== $v"
  IVFTQ_LIB=paper_2605_17415_b200/lib/libivftq_b200_$v.so timeout 120 python scripts/trace_scan.py 10000000 32 96 4096 > gpurun_out/trace_run.log 2>&1
  cp gpurun_out/trace.txt gpurun_out/trace_$v.txt
  python scripts/trace_vq.py gpurun_out/trace.txt
done
