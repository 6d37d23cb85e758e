# operator timings for register-cap variants (HBPDC_MINB 3 / 4 / 5)
make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
for L in libhbpdc_m3.so libhbpdc.so libhbpdc_m5.so; do
  echo "== $L"
  HBPDC_LIB=$PWD/paper_2109_04804_b200/$L timeout 300 python scripts/jvp_only.py 20 2>&1 | tail -4
done
