#!/bin/bash
# KNN float radius bookkeeping + photon tracer pipelining: tests, matrix, full bench line
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_knn.py tests/test_gpu_photon.py tests/test_gpu_train.py tests/test_gpu_renderers.py -m gpu -q -x > $O/pytest_q.log 2>&1; echo "rc=$?" >> $O/pytest_q.log
timeout 900 python tools/bench_knn.py > $O/knn_matrix_q.json 2> $O/knn_matrix_q.err
timeout 900 python bench.py > $O/bench_q.json 2> $O/bench_q.err
