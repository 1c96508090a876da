#!/bin/bash
# KNN probe-cube reach cap: parity + config-3 matrix
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_train.py -m gpu -q -x > $O/pytest_i.log 2>&1; echo "rc=$?" >> $O/pytest_i.log
timeout 900 python tools/bench_knn.py > $O/knn_matrix_i.json 2> $O/knn_matrix_i.err
