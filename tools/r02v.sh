#!/bin/bash
# staged compose A/B + frame hashes (parity and fast) vs the plain compose
export PYTHONPATH=$PWD
O=gpurun_out
for v in cold default; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py parity >> $O/hash_v.txt 2>&1
  python tools/frame_hash.py fast >> $O/hash_v.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh parity cold default cold default > $O/ab_v.txt 2>&1
