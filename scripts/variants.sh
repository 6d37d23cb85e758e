# gpurun helper: op-kernel timings of the default build (+ optional variant builds named
# paper_2109_04804_b200/libhbpdc_<tag>.so passed as arguments)
make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
python scripts/jvp_only.py 10
for v in "$@"; do echo "variant [$v]"; HBPDC_LIB=$PWD/paper_2109_04804_b200/libhbpdc_$v.so python scripts/jvp_only.py 10; done
