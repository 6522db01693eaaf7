# tile warps serialised after the Cholesky chain: off (default) / warps >= 4 / warps >= 10
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
for v in 4 10 0; do
  touch paper_1508_02977_b200/csrc/band.cu
  FFB_NVCC_FLAGS=-DFFB_SERIAL=$v timeout 600 python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/e_build.log 2>&1
  for c in c2 c2 c3; do echo "SERIAL=$v" >> gpurun_out/e_cases.log; timeout 300 python tools/profile_case.py $c >> gpurun_out/e_cases.log 2>&1; done
done
