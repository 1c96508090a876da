#!/bin/bash
# KNN row cursor / float x-range / probe-ring lower bound: parity + matrix; PARITY pipelined-burst tuning A/B
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_tracking.py tests/test_gpu_c2.py -m gpu -q -x > $O/pytest_m.log 2>&1; echo "rc=$?" >> $O/pytest_m.log
timeout 900 python tools/bench_knn.py > $O/knn_matrix_m.json 2> $O/knn_matrix_m.err
bash tools/ab_variants.sh parity default b12 b24 c5 f2 default > $O/ab_m.txt 2>&1
