# round 2, box 21: full chains of c2, c3, c5 with the current library (factor / PCG split)
for c in c2 c3 c5 c2 c3 c5; do timeout 600 python tools/profile_case.py $c >> gpurun_out/r2u.log 2>&1; done
cat gpurun_out/r2u.log
