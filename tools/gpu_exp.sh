# tile solve: owner outputs stored after the broadcast; tests, c2 timings, timeline
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_solve.py tests/test_gpu_ras.py -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest.log
for c in c2 c2 c1; do timeout 300 python tools/profile_case.py $c >> gpurun_out/e_cases.log 2>&1; done
timeout 120 python tools/solve_probe.py c2 >> gpurun_out/e_cases.log 2>&1
FFB_PROFILE=1 timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1; FFB_PROFILE=1 timeout 300 python tools/tile_timeline.py c2 > gpurun_out/t_tl.log 2>&1
