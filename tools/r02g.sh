#!/bin/bash
# KNN bitonic top-k A/B (old full sort vs top-k merge) over the config-3 matrix + KNN parity tests
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_train.py -m gpu -q -x > $O/pytest_g.log 2>&1; echo "rc=$?" >> $O/pytest_g.log
timeout 600 python tools/bench_knn.py > $O/knn_matrix.json 2> $O/knn_matrix.err
PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_old.so timeout 600 python tools/bench_knn.py > $O/knn_matrix_old.json 2> $O/knn_matrix_old.err
