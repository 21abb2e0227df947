#!/bin/bash
# Round profile on one B200: bench lines, ncu launch list, ncu full capture of
# the timed step's kernels.  Usage (under gpurun): bash tools/profile_round.sh TAG
set -u
TAG=${1:-r02a}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
# launch list of the same command in profile mode (cold-cache, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --profile > $OUT/ncu_list.log 2>&1
# full capture: the timed step's traversal, leaf products and C tree (skip the warm-up step)
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"leaf_dmma|traverse_dense|leaf_norm_seg" --launch-skip 12 --launch-count 12 \
  -o $OUT/full -f python bench.py --steps 1 --warmup 1 --profile > $OUT/ncu_full.log 2>&1
for cfg in c1 c3_l3; do
  timeout 600 python bench.py --config $cfg > $OUT/bench_$cfg.log 2>&1
done
