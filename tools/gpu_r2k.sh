# round 2, box 11: extrapolated warm starts between adaptive passes (iteration counts)
for c in c4 c3; do
  for e in none 0.5 1.0 1.5; do
    if [ $e = none ]; then unset FFB_EXTRAP; else export FFB_EXTRAP=$e; fi
    timeout 300 python tools/profile_case.py $c > gpurun_out/r2k_${c}_e$e.log 2>&1
  done
done
unset FFB_EXTRAP
for f in gpurun_out/r2k_*.log; do echo $f; tail -1 $f; done
