#!/usr/bin/env bash
# Round-2 (session e) measurement set on one B200: GPU tests, smoke, the
# default bench line, then ncu evidence of what this session changed -- launch
# lists of the cfg3 row-id lookups (unsorted / sorted ids) and of the cfg5
# probe, full captures of the partition passes, the pair gathers, the fused
# bitvector lookups and the cfg1 small-column scan.  Every profiled command
# runs clean without ncu first.
set -uo pipefail
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r2e}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/gputest_$TAG.txt" 2>&1
tail -2 "$OUT/gputest_$TAG.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1
tail -1 "$OUT/smoke_$TAG.log"
timeout 1500 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"
tail -c 200 "$OUT/bench_$TAG.json"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled -k regex:'bsb::' \
    --csv --log-file "$OUT/launches_lookup_ids_$TAG.csv" python tools/lookup_probe.py 1 28 ids_ \
    > "$OUT/ncu_l1.log" 2>&1
echo "lookup launch list rc=$?"
timeout 600 ncu --metrics $M,smsp__inst_executed.sum --clock-control none --kernel-name-base demangled \
    -k regex:'bsb::' --csv --log-file "$OUT/launches_cfg5_probe_$TAG.csv" \
    python tools/cfg5_probe.py --reps=1 > "$OUT/ncu_l2.log" 2>&1
echo "cfg5 probe launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'pair_|bs_lookup_kernel|vbs_lookup_rows_dec_kernel' -c 14 -o "$OUT/ncu_pairs_$TAG" \
    python tools/lookup_probe.py 1 28 ids_unsorted > "$OUT/ncu_f1.log" 2>&1
echo "pairs full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'lookup_bits_kernel' -c 8 -o "$OUT/ncu_bits_$TAG" \
    python tools/lookup_probe.py 1 28 bits_ > "$OUT/ncu_f2.log" 2>&1
echo "bits full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'bs_scan_small_kernel' -c 2 -o "$OUT/ncu_cfg1_$TAG" \
    python tools/cfg1_probe.py > "$OUT/ncu_f3.log" 2>&1
echo "cfg1 full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'bs_conj_kernel|vbs_dsm_kernel' -c 3 -o "$OUT/ncu_and_$TAG" \
    python tools/cfg5_probe.py --reps=1 > "$OUT/ncu_f4.log" 2>&1
echo "and full rc=$?"
