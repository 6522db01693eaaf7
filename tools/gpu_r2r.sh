# round 2, box 18: full-size parity + multi-rank + RAS with the row-group tile solve, then the bench
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_multi.py tests/test_gpu_ras.py \
  tests/test_gpu_tile_solve.py -x -q > gpurun_out/r2r_tests.log 2>&1
tail -3 gpurun_out/r2r_tests.log
timeout 900 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
cat gpurun_out/r2r_bench.json
