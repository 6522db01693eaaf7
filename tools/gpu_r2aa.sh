# round 2, box 26: where did c5's ring-solve time go? one c5 solve at earlier round-2 commits
# (git worktrees under _wt/, each with its own build) vs HEAD
for i in 1 2; do
  for c in 8016bec 0f4009d c95c64e bd0fe16; do
    echo "$c $(cd _wt/$c && timeout 300 python tools/profile_case.py c5 0 2>&1 | tail -1)" >> gpurun_out/r2aa.log
  done
  echo "HEAD $(timeout 300 python tools/profile_case.py c5 0 2>&1 | tail -1)" >> gpurun_out/r2aa.log
done
cat gpurun_out/r2aa.log
