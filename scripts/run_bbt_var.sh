make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/bbt
C=paper_2109_04804_b200/csrc
for V in "-DTD_E_=512 -DTD_R_=6 -DTD_G_=8 -DTD_C_=2 -DTD_W_=16" "-DTD_E_=512 -DTD_R_=6 -DTD_G_=16 -DTD_C_=1 -DTD_W_=16" "-DTD_E_=1024 -DTD_R_=3 -DTD_G_=8 -DTD_C_=2 -DTD_W_=16" "-DTD_E_=512 -DTD_R_=6 -DTD_G_=12 -DTD_C_=2 -DTD_W_=16"; do
  echo "== $V"
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a $V -I$C scripts/bench_block_tma.cu $C/sstep_tma.cu $C/build/sstep.o $C/build/linalg.o -o /tmp/bbv 2>&1 | grep -i error
  cuobjdump -res-usage /tmp/bbv | grep -A1 dots_tma8 | grep -o "REG:[0-9]*\|LOCAL:[0-9]*"; timeout 120 /tmp/bbv | grep "L=8388608" | cut -c1-100
done 2>&1 | tee gpurun_out/bbt/var.txt
