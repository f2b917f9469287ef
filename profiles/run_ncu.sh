#!/usr/bin/env bash
# Profiling recipe run on the GPU box (see /opt/skills/guides/B200_PROFILING.md).
#   1. plain bench (profile mode) must exit 0 first
#   2. launch list: every kernel with its device time (cold-cache, serialised)
#   3. `ncu --set full` of the four BETWEEN windows of each layout's scan kernel
#      (the first warm-up step; the parity-guard launches are skipped)
# Outputs land in $OUT (gpurun_out/); summaries worth keeping go to profiles/.
set -euo pipefail
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CMD="python bench.py --profile --steps 3 --warmup 1 --no-lookup"
$CMD > "$OUT/profile_plain.log" 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 \
    --csv --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'vbs_ds_kernel' -s 4 -c 4 -o "$OUT/prof_vbs" $CMD > "$OUT/ncu_vbs.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'scan_kernel<.int.0, .bool.1, .bool.0, .bool.0' -s 4 -c 4 -o "$OUT/prof_bs" $CMD \
    > "$OUT/ncu_bs.log" 2>&1
echo done
