#!/bin/bash
# PARITY tracer software pipelining A/B (+ frame hashes)
export PYTHONPATH=$PWD
O=gpurun_out
for v in default pp1 pp6 pp32; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py parity >> $O/hash_l.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh parity default pp1 pp6 pp32 default pp1 > $O/ab_pp.txt 2>&1
