# round 2, box 19: factor per-warp timeline on c4 and c2 (profiling build, on the box only)
FFB_PROFILE=1 timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
FFB_PROFILE=1 timeout 300 python tools/factor_timeline.py c4 > gpurun_out/r2s_ftl_c4.log 2>&1
FFB_PROFILE=1 timeout 300 python tools/factor_timeline.py c2 > gpurun_out/r2s_ftl_c2.log 2>&1
tail -5 gpurun_out/r2s_build.log; head -60 gpurun_out/r2s_ftl_c4.log
