#!/usr/bin/env bash
# One `ncu --set full` capture of a single timed-region kernel of bench.py.
#   KREGEX: demangled-name regex; SKIP: matching launches to skip; NAME: output stem
set -euo pipefail
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CMD="python bench.py --profile --steps 3 --warmup 1 ${BENCH_ARGS:-}"
$CMD > "$OUT/${NAME}_plain.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$KREGEX" -s "${SKIP:-4}" -c "${COUNT:-1}" -o "$OUT/$NAME" $CMD > "$OUT/${NAME}_ncu.log" 2>&1
echo done
