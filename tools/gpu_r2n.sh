# round 2, box 14: A/B of the ring-solve row loop on one box (prev = before the unmasked blocks)
P=$PWD/paper_1508_02977_b200/_variants/libflowfem_b200_prev.so
for i in 1 2; do
  for c in c3 c4; do
    timeout 300 python tools/profile_case.py $c 0 >> gpurun_out/r2n_new_$c.log 2>&1
    FFB_LIB=$P timeout 300 python tools/profile_case.py $c 0 >> gpurun_out/r2n_prev_$c.log 2>&1
  done
done
for f in gpurun_out/r2n_*.log; do echo $f; grep -o "asm [0-9.]* ms" $f; done
