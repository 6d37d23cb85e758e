# K-apply register-cap variants (HBPDC_KAPPLY_MINB 4 / 5 / 6): operator timings + 1-step bench kernels
for L in libhbpdc.so libhbpdc_k5.so libhbpdc_k6.so; do
  echo "== $L"
  HBPDC_LIB=$PWD/paper_2109_04804_b200/$L timeout 300 python scripts/jvp_only.py 20 2>&1 | tail -4
  HBPDC_LIB=$PWD/paper_2109_04804_b200/$L timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('step ms', round(d['ms_per_step'],1), {k: v['ms'] for k, v in d['kernels'].items()})"
done
