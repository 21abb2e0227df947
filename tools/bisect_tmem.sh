# usage: bash tools/bisect_tmem.sh OUTDIR ; alternates default / no-TMEM-stack runs of the 2-process sweep stress
OUT=${1:-gpurun_out/r02m}
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
for cfg in base NOTMEM base_b NOTMEM_b base_c NOTMEM_c; do
  env=""
  case $cfg in NOTMEM*) env="SPAMM_K3_TM_SLOTS=0";; esac
  env $env timeout 400 python tools/stress_sweeps.py --runs 50 --procs 2 > $OUT/$cfg.log 2>&1
  echo "$cfg rc=$? $(grep -o '"n_events": [0-9]*' $OUT/$cfg.log | tr '\n' ' ')" >> $OUT/summary.txt
done
cat $OUT/gpu.txt $OUT/summary.txt
