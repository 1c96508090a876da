#!/bin/bash
# FAST v2 (ready queue + cell bursts + parked collisions) A/B + frame hashes vs v1
export PYTHONPATH=$PWD
O=gpurun_out
for v in v1 default c7; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py fast >> $O/hash_w.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh fast v1 default c7 c6 f2 r2 b8 b32 v1 default > $O/ab_w.txt 2>&1
