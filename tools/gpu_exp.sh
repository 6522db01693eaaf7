# L1 prefetch of the look-ahead block: on (default) / off; c2/c3 timings, c2 timeline
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest.log
for v in 1 0; do
  touch paper_1508_02977_b200/csrc/band.cu
  FFB_NVCC_FLAGS=-DFFB_KKPF=$v timeout 600 python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/e_build.log 2>&1
  for c in c2 c2 c3; do echo "KKPF=$v" >> gpurun_out/e_cases.log; timeout 300 python tools/profile_case.py $c >> gpurun_out/e_cases.log 2>&1; done
done
bash tools/gpu_ftl.sh c2
