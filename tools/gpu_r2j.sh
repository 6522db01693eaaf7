# round 2, box 10: ring-solve knobs on c4 with the persistent queue (stages, row cost)
for st in 2 3 4; do FFB_STAGES=$st timeout 300 python tools/profile_case.py c4 0 > gpurun_out/r2j_st$st.log 2>&1; done
for rc in 0 8 16 32; do FFB_ROW_COST=$rc timeout 300 python tools/profile_case.py c4 0 > gpurun_out/r2j_rc$rc.log 2>&1; done
for f in gpurun_out/r2j_*.log; do echo $f; tail -1 $f; done
