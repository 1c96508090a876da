#!/bin/bash
# FAST DDA next-cell prefetch A/B (+ frame hashes)
export PYTHONPATH=$PWD
O=gpurun_out
for v in np default; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py fast >> $O/hash_r.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh fast np default np default > $O/ab_r.txt 2>&1
