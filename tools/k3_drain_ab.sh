# A/B of K3's final-wave ticket policy (SPAMM_K3_DRAIN) on c2 and c3 lambda=2
for v in 0 1 2 0 1 2; do
  for cfg in c2 c3_l2; do
    SPAMM_K3_DRAIN=$v timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('drain=$v $cfg', round(d['value'],3), round(d['roofline']['frac'],4))"
  done
done
