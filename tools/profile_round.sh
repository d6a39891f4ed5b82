#!/usr/bin/env bash
# One GPU-box pass that regenerates the round's measured artifacts:
#   bench line (ours + reference arm), the ncu launch list of the bench
#   command, and one `ncu --set full` capture of the render kernel.
# Usage (from the repo root, on a B200):  bash tools/profile_round.sh <tag>
# Outputs land in gpurun_out/<tag>_*; copy what is judged into profiles/.
set -u
tag=${1:-round}
out=gpurun_out
mkdir -p "$out"
python bench.py > "$out/${tag}_bench.json" 2> "$out/${tag}_bench.err" || echo "bench failed"
python bench.py --impl reference --steps 3 --warmup 1 > "$out/${tag}_bench_reference.json" \
  2> "$out/${tag}_bench_reference.err" || echo "reference arm failed"
# launch list of the same bench command (serialised, cold caches: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$out/${tag}_launches.csv" \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > "$out/${tag}_ncu_list.log" 2>&1 \
  || echo "ncu launch list failed"
# one full capture of a steady-state render launch
ncu --set full --import-source on --clock-control none -k regex:render_step -s 8 -c 1 \
  -o "$out/${tag}_render_full" \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > "$out/${tag}_ncu_full.log" 2>&1 \
  || echo "ncu full capture failed"
tail -c 2000 "$out/${tag}_bench.json"
