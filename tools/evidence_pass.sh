#!/bin/bash
# Evidence pass (one gpurun call): full GPU suite, the driver's bench
# lines (ours, reference arm, C4, C5), the launch list, and ncu captures of
# every hot kernel, summarised on the box.  Timing numbers come from bench.py only.
export PYTHONPATH=$PWD
O=gpurun_out
mkdir -p $O/prof
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/prof/gpu.txt 2>&1
nproc > $O/prof/host.txt; grep -m1 "model name" /proc/cpuinfo >> $O/prof/host.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/prof/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/prof/pytest_gpu.log
timeout 900 python bench.py > $O/prof/bench.json.txt 2> $O/prof/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/prof/bench_ref.json.txt 2> $O/prof/bench_ref.err
timeout 600 python bench.py --config c4 --no-extras --no-cpu-baseline --steps 10 > $O/prof/bench_c4.json.txt 2> $O/prof/bench_c4.err
timeout 600 python bench.py --config c5 --no-extras --no-cpu-baseline --steps 20 > $O/prof/bench_c5.json.txt 2> $O/prof/bench_c5.err
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/prof/launches_frame.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --no-fast > /dev/null 2>&1
python tools/launch_shares.py $O/prof/launches_frame.csv > $O/prof/launch_shares.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"k_render_trace_parity|k_field_encode|k_field_mlp|k_compose" -s 4 -c 4 \
    -o $O/frame_par python tools/profile_frame.py --mode parity --frames 3 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:"k_render_trace_fast" -s 1 -c 1 \
    -o $O/trace_fast python tools/profile_frame.py --mode fast --frames 2 > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"k_knn_query_sel" -c 1 \
    -o $O/knn_sel python tools/knn_traced_probe.py uniform inf > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"k_knn_query_cta|k_train_(fwd|bwd|adam|wgrad|scatter)|k_trace_photons" -s 2 -c 7 \
    -o $O/train_full python tools/bench_train.py --steps 2 --photons 200000 > /dev/null 2>&1
for r in frame_par trace_fast knn_sel train_full; do
  python tools/ncu_summary.py $O/$r.ncu-rep $O/prof/$r > /dev/null 2>&1
done
ncu -i $O/frame_par.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_render_trace_parity > $O/par_src.csv 2>/dev/null
python tools/ncu_lines.py $O/par_src.csv 656400000 50 > $O/prof/lines_trace_parity.txt 2>&1
ncu -i $O/knn_sel.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_knn_query_sel > $O/knn_src.csv 2>/dev/null
python tools/ncu_lines.py $O/knn_src.csv 1048576 40 > $O/prof/lines_knn_sel.txt 2>&1
python tools/ncu_hotspots.py $O/frame_par.ncu-rep k_field_mlp > $O/prof/hot_field_mlp.md 2>&1
python tools/ncu_hotspots.py $O/trace_fast.ncu-rep k_render_trace_fast > $O/prof/hot_trace_fast.md 2>&1
# only the summaries travel back (gpurun_out is capped at 64 MiB)
rm -f $O/*.ncu-rep $O/par_src.csv $O/knn_src.csv
ls -la $O/prof
