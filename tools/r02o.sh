#!/bin/bash
# PARITY tracer: two steps in flight A/B (+ frame hashes)
export PYTHONPATH=$PWD
O=gpurun_out
for v in default d2 d2c4 d2c6; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py parity >> $O/hash_o.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh parity default d2 d2c4 d2c6 default d2 > $O/ab_o.txt 2>&1
