# operator timings for CTA-size variants (HBPDC_CTA_THREADS 64 / 128 / 256: 1 / 2 / 4 N=7 elements per CTA)
for L in libhbpdc_t64.so libhbpdc.so libhbpdc_t256.so; do
  echo "== $L"
  HBPDC_LIB=$PWD/paper_2109_04804_b200/$L timeout 300 python scripts/jvp_only.py 20 2>&1 | tail -4
done
