#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the launch list, then one full
# capture per kernel of interest (all ncu runs of one gpurun call count as one ncu use).
CMD="python bench.py --views 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stage-events --no-c3"
KERNELS=${KERNELS:-"k_composite_tc k_bin_place k_tile_split k_bin_count k_sort_pass k_sort_digits k_project k_unproject_write"}
TAG=${TAG:-prof}
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for k in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:"^.*${k}" -s ${SKIP:-5} -c 1 -o gpurun_out/${TAG}_${k} $CMD > gpurun_out/ncu_${k}.log 2>&1
  echo "$k rc=$?"
done
