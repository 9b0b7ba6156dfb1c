timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cfg3 or bf16 or cfg2" 2>&1 | tail -4
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
tail -n 2 gpurun_out/bench3.err
