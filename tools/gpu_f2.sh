for e in "" "FFB_FSPLIT=1" "FFB_NB=16" "FFB_FACTOR_MMA=0" "FFB_FCLUSTER=8" "FFB_FCLUSTER=2"; do
  echo "== $e"; env $e timeout 120 python tools/profile_case.py c2 2>&1 | tail -1
done > gpurun_out/f2.log 2>&1
cat gpurun_out/f2.log
