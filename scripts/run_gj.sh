make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
for L in libhbpdc.so libhbpdc_g1.so libhbpdc_g2.so; do
  HBPDC_LIB=$PWD/paper_2109_04804_b200/$L timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$L', d['ms_per_step'], d['kernels']['build'])"
done
