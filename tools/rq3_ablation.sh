#!/bin/bash
# RQ3 analog (Table 4): the host module's computation-free handling on vs off.
#   on  (default): zero-copy exits (the next fused block reads survivors through the row list),
#                  in-place gates (executed rows rewritten through the list, skipped rows untouched)
#   off (DYCL_NO_ZERO_COPY=1 DYCL_NO_INPLACE=1): identity copies materialised -- exits gather the
#                  survivors, gates gather the executed rows and merge both branches back
mkdir -p gpurun_out
: > gpurun_out/rq3.jsonl
run() {  # tag env... -- args
  tag=$1; shift
  env "$@" > gpurun_out/rq3_$tag.json 2> gpurun_out/rq3_$tag.err
  tail -1 gpurun_out/rq3_$tag.json | python -c "import json,sys; l=json.loads(sys.stdin.read()); l['ablation']='$tag'; print(json.dumps(l))" >> gpurun_out/rq3.jsonl
}
for c in 2 3; do
  run c${c}_on timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline
  run c${c}_off DYCL_NO_ZERO_COPY=1 DYCL_NO_INPLACE=1 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline
done
run c3r_on timeout 600 python bench.py --config 3 --rnn-gates --steps 30 --warmup 5 --no-cpu-baseline
run c3r_off DYCL_NO_ZERO_COPY=1 DYCL_NO_INPLACE=1 timeout 600 python bench.py --config 3 --rnn-gates --steps 30 --warmup 5 --no-cpu-baseline
run c5_on timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline
run c5_off DYCL_NO_ZERO_COPY=1 DYCL_NO_INPLACE=1 timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline
wc -l gpurun_out/rq3.jsonl
