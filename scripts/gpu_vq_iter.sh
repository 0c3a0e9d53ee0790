# scan_vq iteration: parity tests, C3/C2-shape scan timing, trace of CTA 0
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 200 python scripts/scan_exp.py 10000000 32 96 4096 2>&1 | tail -1
timeout 200 python scripts/scan_exp.py 1000000 64 128 1024 2>&1 | tail -1
bash scripts/gpu_vq_trace.sh 10000000 32 96 4096
