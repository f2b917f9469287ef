#!/usr/bin/env bash
# Round-2 measurement set on one B200 (run from the repo root on the GPU box):
# GPU tests, smoke, the default bench line, then the ncu evidence --
# launch list of the cfg5 step (eager, one step), full captures of the cfg5
# kernels on one segment, and the cfg2 / lookup captures.
set -uo pipefail
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r2}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/gputest_$TAG.log" 2>&1
tail -2 "$OUT/gputest_$TAG.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1
tail -1 "$OUT/smoke_$TAG.log"
timeout 1500 python bench.py > "$OUT/bench_$TAG.log" 2>&1
tail -c 300 "$OUT/bench_$TAG.log"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k regex:'bs_|vbs_|bsb::' \
    --csv --log-file "$OUT/launches_bench_$TAG.csv" \
    python bench.py --profile --no-graph --steps 1 --warmup 1 --no-extra --no-cpu-baseline \
    > "$OUT/ncu_launches_bench_$TAG.log" 2>&1
echo "launch list rc=$?"
TAG=$TAG COUNT=27 timeout 1200 bash profiles/run_ncu_cfg5.sh > "$OUT/ncu_cfg5_$TAG.log" 2>&1
echo "cfg5 full rc=$?"
