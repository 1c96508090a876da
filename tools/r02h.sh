#!/bin/bash
# MLP sub-chunk pipeline (chunk width A/B) + KNN bracketed radius search
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_knn.py tests/test_gpu_c2.py tests/test_gpu_train.py -m gpu -q -x > $O/pytest_h.log 2>&1; echo "rc=$?" >> $O/pytest_h.log
bash tools/ab_variants.sh fast old default cw16 cw64 > $O/ab_cw.txt 2>&1
timeout 900 python tools/bench_knn.py > $O/knn_matrix_h.json 2> $O/knn_matrix_h.err
