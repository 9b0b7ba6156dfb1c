#!/bin/bash
# Every workload through bench.py (one JSON line each) -> gpurun_out/bench_all.jsonl
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
: > gpurun_out/bench_all.jsonl
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -1 gpurun_out/bench_$tag.json >> gpurun_out/bench_all.jsonl; }
run c5 --config 5
run c2 --config 2
run c1 --config 1
run c3 --config 3
run c3r --config 3 --rnn-gates
run c4 --config 4 --steps 10
run cap --config 4 --caption --steps 10
run ref5 --impl reference --config 5 --steps 3 --warmup 3
wc -l gpurun_out/bench_all.jsonl
