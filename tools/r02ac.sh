#!/bin/bash
# K7c (K=1024 training targets) source-level profile on the bench_train workload
export PYTHONPATH=$PWD
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_knn_query_cta" -s 2 -c 1 \
    -o $O/k7c python tools/bench_train.py --steps 2 > $O/k7c.log 2>&1
ncu -i $O/k7c.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_knn_query_cta > $O/k7c_src.csv 2>/dev/null
python tools/ncu_summary.py $O/k7c.ncu-rep $O/k7c_sum > /dev/null 2>&1
python tools/ncu_lines.py $O/k7c_src.csv 65536 60 > $O/k7c_lines.txt 2>&1
rm -f $O/k7c.ncu-rep $O/k7c_src.csv
