# round 2 (re-entry), box 10: factor build-time knobs on c4 (one full factorisation + first solve; factor ms)
for v in "" ZSPLIT_1 ZSPLIT_4 RG_1 RG_4 KKPF_0 ""; do
  if [ -z "$v" ]; then unset FFB_LIB; else export FFB_LIB=$PWD/paper_1508_02977_b200/_variants/lib_$v.so; fi
  echo "== ${v:-default}"; timeout 300 python tools/profile_case.py c4 0 2>&1 | tail -1 | cut -c1-120
done
