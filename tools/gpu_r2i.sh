# round 2, box 9: factor cluster size on c4 (more lines in flight when the factor is latency-bound)
for fc in 4 2 1; do
  FFB_FCLUSTER=$fc timeout 600 python tools/profile_case.py c4 > gpurun_out/r2i_fc$fc.log 2>&1
  FFB_FCLUSTER=$fc timeout 600 python tools/profile_case.py c4 >> gpurun_out/r2i_fc$fc.log 2>&1
done
for fc in 4 2 1; do echo "FCLUSTER $fc"; cat gpurun_out/r2i_fc$fc.log; done
timeout 900 python -m pytest tests/test_gpu_factor_variants.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2i_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2i_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r2i_factor_c4 python tools/profile_case.py c4 0 > gpurun_out/r2i_ncu_factor.log 2>&1
tail -3 gpurun_out/r2i_tests.log
