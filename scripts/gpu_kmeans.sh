# device k-means: parity tests, then the refresh-sized timing (411k x 4096 x 96)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "kmeans or train_partition or Refresh or refresh" 2>&1 | tail -15
timeout 300 python scripts/kmeans_time.py 2>&1 | tail -3
