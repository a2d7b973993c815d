#!/bin/bash
# Profiling capture for profiles/ (run on the B200 box from the repo root):
#   gpurun --timeout 1500 -- 'bash tools/capture_profiles.sh r2'
# 1. bench.py (1 lane, no profiler) -> gpurun_out/<tag>_bench.json
# 2. launch list of two homogenizations, graph-free (tools/gmg_one.py --profiling)
# 3. ncu --set full of the level-0 apply, the level-0 sweep, the update kernel and the field kernel
set -u
T=${1:-r2}
O=gpurun_out
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file $O/${T}_launches.csv python tools/gmg_one.py --profiling > $O/${T}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'brick_apply_kernel' -c 2 \
    -o $O/${T}_apply -f python tools/gmg_one.py > $O/${T}_ncu_apply.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'brick_sweep_kernel|update_kernel|field_samples_kernel|prolong_kernel|restrict_kernel|coarsest_cluster_kernel|level_sweep3_kernel|coarse_warp_sweep_kernel' -c 14 \
    -o $O/${T}_kernels -f python tools/gmg_one.py > $O/${T}_ncu_kernels.log 2>&1
echo done
