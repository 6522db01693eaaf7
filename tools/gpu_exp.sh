# A_RK tiles on DMMA (default) vs FFMA: tests on the default, c2/c3 timings, c2 timeline
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_solve.py tests/test_gpu_factor_variants.py -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest.log
for v in 1 0; do
  touch paper_1508_02977_b200/csrc/band.cu
  FFB_NVCC_FLAGS=-DFFB_ARK_MMA=$v timeout 600 python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/e_build.log 2>&1
  for c in c2 c2 c3; do echo "ARK_MMA=$v" >> gpurun_out/e_cases.log; timeout 300 python tools/profile_case.py $c >> gpurun_out/e_cases.log 2>&1; done
done
touch paper_1508_02977_b200/csrc/band.cu
bash tools/gpu_ftl.sh c2
