# round 2 (re-entry), box 7: factor cluster size on c4 / c3 / c5 (full adaptive chains; factor ms is the sum of all factorisations)
for c in c4 c3; do
  for fc in 4 2 1; do
    echo "== $c FFB_FCLUSTER=$fc"; FFB_FCLUSTER=$fc timeout 300 python tools/profile_case.py $c 2>&1 | tail -1
  done
done
echo "== c5 FFB_FCLUSTER=4"; FFB_FCLUSTER=4 timeout 300 python tools/profile_case.py c5 2>&1 | tail -1
echo "== c5 default (8)"; timeout 300 python tools/profile_case.py c5 2>&1 | tail -1
