# scan_vq iteration: parity tests, then C3-shape scan timing (default + bound builds), then traces
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q 2>&1 | tail -3
timeout 200 python scripts/scan_exp.py 10000000 32 96 4096 2>&1 | tail -1
for v in ${VARIANTS:-noepi nopush nodec_noepi}; do IVFTQ_LIB=paper_2605_17415_b200/lib/libivftq_b200_exp_$v.so timeout 200 python scripts/scan_exp.py 10000000 32 96 4096 2>&1 | tail -1; done
IVFTQ_SCAN_VQ=1 bash scripts/gpu_trace_exp.sh
