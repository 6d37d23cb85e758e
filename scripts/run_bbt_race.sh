make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
C=paper_2109_04804_b200/csrc
for V in "-DTF_E_=512 -DTF_R_=6 -DTF_FENCE=fence_proxy_async_smem()" "-DTF_E_=256 -DTF_R_=12" "-DTF_E_=512 -DTF_R_=5"; do
  echo "== $V"
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a $V -I$C scripts/bench_block_tma.cu $C/sstep_tma.cu $C/build/sstep.o $C/build/linalg.o -o /tmp/bbr 2>&1 | grep -i error
  for i in 1 2 3; do timeout 120 /tmp/bbr | grep "fused\|check" | grep -v "e-1[3-7] W diff" | cut -c1-150; done
done
