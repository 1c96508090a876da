#!/bin/bash
# KNN geometric probe: parity + matrix; PARITY log table in smem A/B (+ frame hashes)
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py -m gpu -q -x > $O/pytest_j.log 2>&1; echo "rc=$?" >> $O/pytest_j.log
timeout 900 python tools/bench_knn.py > $O/knn_matrix_j.json 2> $O/knn_matrix_j.err
for v in default lg1; do
  if [ $v = default ]; then unset PF_LIBPFGPU; else export PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_$v.so; fi
  python tools/frame_hash.py parity >> $O/hash_j.txt 2>&1
done
unset PF_LIBPFGPU
bash tools/ab_variants.sh parity default lg1 default lg1 > $O/ab_lg.txt 2>&1
