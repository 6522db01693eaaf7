# c2 factor timeline (profiling build)
FFB_PROFILE=1 timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
FFB_PROFILE=1 timeout 300 python tools/factor_timeline.py ${1:-c2} > gpurun_out/e_ftl.log 2>&1
