#!/bin/bash
# KNN on the traced map: launch list + ncu source profile of the select kernel
export PYTHONPATH=$PWD
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_knn|k_make" --csv \
   --log-file $O/knn_traced_launches.csv python tools/knn_traced_probe.py traced inf > $O/knn_probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_knn_query_sel" -c 1 \
   -o $O/knn_traced python tools/knn_traced_probe.py traced inf >> $O/knn_probe.log 2>&1
ncu -i $O/knn_traced.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_knn_query_sel > $O/knn_traced_src.csv 2>/dev/null
python tools/ncu_summary.py $O/knn_traced.ncu-rep $O/knn_traced_sum > /dev/null 2>&1
