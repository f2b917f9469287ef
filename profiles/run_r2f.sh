#!/usr/bin/env bash
# Final round-2 set on one B200: GPU tests, smoke, the default bench line, the
# reference arm, then the ncu launch list of the bench command's cfg5 step
# (eager launches, one step; build / parity kernels included, the timed step's
# kernels last) for the per-kernel share of the step.
set -uo pipefail
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r2f}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/gputest_$TAG.txt" 2>&1
tail -2 "$OUT/gputest_$TAG.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1
tail -1 "$OUT/smoke_$TAG.log"
timeout 1500 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"
tail -c 200 "$OUT/bench_$TAG.json"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref_$TAG.json" 2> "$OUT/bench_ref_$TAG.err"
tail -c 300 "$OUT/bench_ref_$TAG.json"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k regex:'bs_|vbs_|bsb::' \
    --csv --log-file "$OUT/launches_bench_$TAG.csv" \
    python bench.py --profile --no-graph --steps 1 --warmup 1 --no-extra --no-cpu-baseline \
    > "$OUT/ncu_launches_bench_$TAG.log" 2>&1
echo "launch list rc=$?"
