timeout 900 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
tail -n 2 gpurun_out/bench2.err
