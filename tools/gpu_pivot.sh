# pivot microbench (alone / with 14 busy warps) + the c2 factor timeline (profiling build)
set -x
cd tools/microbench && timeout 60 ./pivot > ../../gpurun_out/pivot_mb.log 2>&1; cd ../..
FFB_PROFILE=1 timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof_build.log 2>&1
FFB_PROFILE=1 timeout 300 python tools/factor_timeline.py c2 > gpurun_out/ftl_c2.log 2>&1
