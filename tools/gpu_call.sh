timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cfg4 or cfg1 or dense or conv_kernel" 2>&1 | tail -2
timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
