python scripts/trace_scan.py 10000000 32 96 4096 > gpurun_out/trace_c3.log 2>&1; python scripts/trace_stats.py gpurun_out/trace.txt > gpurun_out/trace_c3_stats.txt 2>&1; cp gpurun_out/trace.txt gpurun_out/trace_c3.txt
B="python bench.py --steps 1 --warmup 3 --no-parity --no-cpu-baseline"
$B > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:scan_tc_kernel -s 6 -c 1 -o gpurun_out/scan_c3 $B > gpurun_out/ncu_c3.log 2>&1
tail -3 gpurun_out/ncu_c3.log; cat gpurun_out/trace_c3_stats.txt
