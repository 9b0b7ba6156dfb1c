#!/bin/bash
# which commit broke test_cfg2_rebalance_on_equals_off[2-equal-device]? run it against older builds
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
: > gpurun_out/bisect.txt
for lib in bisect/lib_57579ae.so bisect/lib_4535e33.so bisect/lib_8ae6179.so paper_2307_04963_b200/libdycl.so; do
  r=$(timeout 300 python -c "
import sys
import paper_2307_04963_b200.dycl as D
D.LIB_PATH='$lib'
import pytest
sys.exit(pytest.main(['-q','-m','gpu','tests/test_gpu_multi.py','-k','test_cfg2_rebalance_on_equals_off and 2-equal-device','-p','no:cacheprovider']))
" 2>&1 | tail -1)
  echo "$lib: $r" >> gpurun_out/bisect.txt
done
cat gpurun_out/bisect.txt
