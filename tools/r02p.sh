#!/bin/bash
# KNN same-box A/B (pre-top-k vs current) + ncu source profile of the select kernel on the uniform map
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 python tools/bench_knn.py > $O/knn_matrix_p.json 2> $O/knn_matrix_p.err
PF_LIBPFGPU=$PWD/paper_2304_07338_b200/libpfgpu_kold.so timeout 900 python tools/bench_knn.py > $O/knn_matrix_pold.json 2> $O/knn_matrix_pold.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_knn_query_sel" -c 1 \
   -o $O/knn_uniform python tools/knn_traced_probe.py uniform inf > $O/knn_probe_p.log 2>&1
ncu -i $O/knn_uniform.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_knn_query_sel > $O/knn_uniform_src.csv 2>/dev/null
python tools/ncu_summary.py $O/knn_uniform.ncu-rep $O/knn_uniform_sum > /dev/null 2>&1
