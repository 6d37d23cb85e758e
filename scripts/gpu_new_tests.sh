make -C paper_2109_04804_b200/csrc -j8 > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/nt
timeout 1200 python -m pytest tests -m gpu -x -q -k "glf or mach or sstep_pipeline or bjext_h" > gpurun_out/nt/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/nt/pytest.log
timeout 900 python scripts/iteration_study.py > gpurun_out/nt/iteration_study.md 2> gpurun_out/nt/it.err; echo "it rc=$?"
bash scripts/run_minb.sh 2>&1 | tee gpurun_out/nt/minb.txt
