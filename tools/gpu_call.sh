timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cfg4 or nhwc or cfg5 or cfg1" 2>&1 | tail -3
timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
DYCL_S2S_GEMM=0 timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4b.json 2>> gpurun_out/bench4.err
timeout 300 python tools/step_profile5.py 2048 2 > gpurun_out/prof5_nhwc.json 2> gpurun_out/prof5.err
