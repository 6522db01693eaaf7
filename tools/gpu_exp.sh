# tile solve: non-volatile mapa (hoistable); tests, c1/c2 application timings
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_solve.py tests/test_gpu_ras.py -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest.log
for c in c2 c1 c2 c1; do timeout 200 python tools/solve_probe.py $c >> gpurun_out/e_cases.log 2>&1; done
