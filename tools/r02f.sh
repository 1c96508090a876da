#!/bin/bash
# training resume + KNN config-3 matrix (Stream::Train queries; uniform / clustered / traced maps; r_max inf/0.05/0.25)
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_capi.py tests/test_gpu_knn.py -m gpu -q -x > $O/pytest_f.log 2>&1; echo "rc=$?" >> $O/pytest_f.log
timeout 600 python tools/bench_knn.py > $O/knn_matrix.json 2> $O/knn_matrix.err
