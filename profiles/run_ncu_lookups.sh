#!/usr/bin/env bash
# ncu --set full of the fused bitvector lookups (cfg3: 1 % and 20 %
# selections, ByteSlice and PP-VBS) and the row-id lookups, after the plain
# probe exits 0.  Outputs in $OUT.
set -euo pipefail
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
python tools/lookup_probe.py 3 28 > "$OUT/lookup_plain.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'lookup_bits_kernel|bs_lookup_kernel|vbs_lookup_rows_dec_kernel' -c 16 \
    -o "$OUT/prof_lookups" python tools/lookup_probe.py 1 28 > "$OUT/ncu_lookups.log" 2>&1
echo done
