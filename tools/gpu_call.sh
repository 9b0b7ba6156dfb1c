timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cfg2 or cfg3 or bf16 or permutation or run_host or empty" 2>&1 | tail -5 > gpurun_out/t2.log
python tools/ts_probe.py 2 > gpurun_out/ts2.txt 2>&1; python tools/ts_probe.py 1 > gpurun_out/ts1.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
cat gpurun_out/t2.log; head -4 gpurun_out/ts2.txt; head -4 gpurun_out/ts1.txt; tail -2 gpurun_out/bench2.err
