#!/usr/bin/env bash
# cfg5 profiling recipe (GPU box): one 2^29-row segment per column via
# tools/cfg5_probe.py.  1) plain run must exit 0; 2) launch list of every
# kernel (cold-cache, serialised); 3) ncu --set full of the scan kernels of
# the five queries (u0/u1 ByteSlice, z0/z1 PP-VBS, the AND chain's legs).
set -euo pipefail
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r2}
mkdir -p "$OUT"
CMD="python tools/cfg5_probe.py --reps=1"
$CMD > "$OUT/cfg5_probe_plain_$TAG.log" 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled \
    --csv --log-file "$OUT/launches_cfg5_$TAG.csv" $CMD > "$OUT/ncu_launches_cfg5_$TAG.log" 2>&1
# the timed launches: skip the build / parity kernels, capture each query's scan
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'scan_kernel|vbs_ds_kernel|bs_conj_kernel' -s ${SKIP:-0} -c ${COUNT:-40} -o "$OUT/prof_cfg5_$TAG" \
    $CMD > "$OUT/ncu_full_cfg5_$TAG.log" 2>&1
echo done
