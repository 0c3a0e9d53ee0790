for v in libivftq_b200_sleep0.so libivftq_b200.so libivftq_b200_sleep200.so; do
  IVFTQ_SCAN_VQ=1 IVFTQ_LIB=paper_2605_17415_b200/lib/$v timeout -k 5 120 python scripts/scan_exp.py 10000000 32 96 4096 2>&1 | tail -1
done
