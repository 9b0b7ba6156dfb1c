timeout 900 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
