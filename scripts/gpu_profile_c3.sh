# C3 evidence: the launch list of the timed bench steps and one ncu --set full of the scan
B="python bench.py --steps 3 --warmup 3 --no-parity --no-cpu-baseline"
timeout -k 5 300 $B > gpurun_out/plain_p.log 2>&1 && IVFTQ_PROFILE_STEPS=1 timeout -k 5 500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_steps.csv $B > gpurun_out/ncu_steps.log 2>&1
S="python scripts/scan_exp.py 10000000 32 96 4096"
timeout -k 5 200 $S > gpurun_out/plain_s.log 2>&1 && timeout -k 5 400 ncu --set full --clock-control none --import-source on -k regex:scan_vq_kernel -s 2 -c 1 -o gpurun_out/vq_c3_full $S > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
