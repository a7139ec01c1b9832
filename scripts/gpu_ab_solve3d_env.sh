# same-box A/B of the 3D solve over env settings ($COMBOS lines), cfg4 model at n^3.
for rep in 1 2; do
echo "$COMBOS" | while read -r envs; do
  for spec in ${SPECS:-"128,8,c128" "128,8,c64"}; do
    IFS=, read n b d <<< "$spec"
    env $envs timeout 300 python scripts/solve3d.py $n $b $d 2 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$envs', d['n'], d['dtype'], d['ms'], d['GBps'], 'L1 arnoldi', d['levels'].get('1',{}).get('arnoldi'))"
  done
done; done
