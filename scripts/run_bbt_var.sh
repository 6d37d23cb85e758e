make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
C=paper_2109_04804_b200/csrc
for V in "-DTF_W_=8" "-DTF_W_=16" "-DTF_W_=16 -DTF_MAXT_=16"; do
  echo "== $V"
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a $V -I$C scripts/bench_block_tma.cu $C/sstep_tma.cu $C/build/sstep.o $C/build/linalg.o -o /tmp/bbv 2>&1 | grep -i error
  timeout 200 /tmp/bbv | grep "L=8388608.*fused\|check" | cut -c1-120
done
