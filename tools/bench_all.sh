#!/bin/bash
# All five configs through bench.py (one JSON line each) -> gpurun_out/bench_all.jsonl
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
for c in 2 1 3 4 5; do
  extra=""
  if [ "$c" = "5" ]; then extra="--steps 5 --warmup 3"; fi
  timeout 900 python bench.py --config $c $extra > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  tail -1 gpurun_out/bench_c$c.json >> gpurun_out/bench_all.jsonl
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -1 gpurun_out/bench_ref.json >> gpurun_out/bench_all.jsonl
