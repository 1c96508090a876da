#!/bin/bash
# FAST tracer ready-queue A/B + frame hashes vs the previous kernel
export PYTHONPATH=$PWD
O=gpurun_out
for v in old default; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py fast >> $O/hash_e.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh fast old default r2 r4 r16 c7 > $O/ab_fast.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_render.py tests/test_gpu_configs.py -m gpu -q -x > $O/pytest_e.log 2>&1; echo "rc=$?" >> $O/pytest_e.log
