mkdir -p gpurun_out/r02o
for v in 8 0 8 0; do
  for cfg in c2 c3_l2; do
    SPAMM_K3_TM_SLOTS=$v timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --no-extra > gpurun_out/r02o/tm${v}_$cfg.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/r02o/tm${v}_$cfg.json').read().strip().splitlines()[-1]); print('tm=$v $cfg', round(d['value'],3), round(d['roofline']['frac'],4))" >> gpurun_out/r02o/summary.txt
  done
done
cat gpurun_out/r02o/summary.txt
