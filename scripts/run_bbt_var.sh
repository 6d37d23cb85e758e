make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/bbt
C=paper_2109_04804_b200/csrc
for V in "-DTF_E_=512 -DTF_R_=5" "-DTF_E_=512 -DTF_R_=4" "-DTF_E_=256 -DTF_R_=6"; do
  echo "== $V"
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a $V -I$C scripts/bench_block_tma.cu $C/sstep_tma.cu $C/build/sstep.o $C/build/linalg.o -o /tmp/bbv 2>&1 | grep -i error
  timeout 120 /tmp/bbv | grep "fused\|check\|bad row" | cut -c1-130
done 2>&1 | tee gpurun_out/bbt/var.txt
