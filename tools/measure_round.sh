#!/usr/bin/env bash
# The round's measured artifacts (no profiler): headline bench line + the
# reference arm, BASELINE configs 1-3, the large-pack variant, the sweep.
# usage (GPU box, repo root): bash tools/measure_round.sh <tag>
tag=${1:-r2}
o=gpurun_out
export PYTHONDONTWRITEBYTECODE=1
python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err || echo "bench failed"
python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err
for c in "1 HalfCheetah 1 none" "2 Ant 1024 color" "3 Walker2d 4096 video"; do
  set -- $c
  python bench.py --model $2 --envs $3 --mode $4 > $o/${tag}_bench_config$1.json 2> $o/${tag}_bench_config$1.err
  python bench.py --impl reference --model $2 --envs $3 --mode $4 --steps 3 --warmup 1 > $o/${tag}_bench_config$1_reference.json 2>> $o/${tag}_bench_config$1.err
done
python bench.py --pack-videos 1024 --no-cpu-baseline > $o/${tag}_bench_largepack.json 2> $o/${tag}_bench_largepack.err
python tools/sweep.py --out $o/${tag}_sweep > $o/${tag}_sweep.log 2>&1
for f in $o/${tag}_bench*.json; do echo "$f: $(grep -o '"value": [0-9.e+]*' $f | head -1)"; done
