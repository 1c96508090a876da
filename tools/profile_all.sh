#!/bin/bash
# One GPU-box pass that refreshes the evidence under profiles/ (run via gpurun;
# outputs land in gpurun_out/).  Timing numbers come from bench.py only.
set -x
export PYTHONPATH=$PWD
O=gpurun_out
python bench.py > $O/bench.json 2> $O/bench.err
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/launches_frame.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
$NCU --set full --import-source on -k regex:"k_render_trace_fast" -s 2 -c 1 \
    -o $O/trace_full python tools/profile_frame.py --frames 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:"k_field_encode|k_field_mlp" -s 4 -c 2 \
    -o $O/frame_full python tools/profile_frame.py --frames 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:"k_render_pt|k_knn_query_sel" -s 1 -c 2 \
    -o $O/renderers_full python tools/profile_renderers.py > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_knn_query_sel -s 2 -c 1 -o $O/knn_sel_full \
    python tools/bench_knn.py > /dev/null 2>&1
$NCU --set full --import-source on -k regex:"k_knn_query_cta|k_train_(fwd|bwd|adam|wgrad)" -s 8 -c 5 \
    -o $O/train_full python tools/bench_train.py --steps 2 --photons 200000 > /dev/null 2>&1
# summarise on the box (reports are too large to ship back)
mkdir -p $O/prof
for r in trace_full frame_full renderers_full knn_sel_full train_full; do
  python tools/ncu_summary.py $O/$r.ncu-rep $O/prof/$r > /dev/null 2>&1
done
python tools/ncu_hotspots.py $O/trace_full.ncu-rep k_render_trace_fast > $O/prof/hot_trace_fast.md
python tools/ncu_hotspots.py $O/frame_full.ncu-rep k_field_mlp > $O/prof/hot_field_mlp.md
python tools/ncu_hotspots.py $O/renderers_full.ncu-rep k_render_pt > $O/prof/hot_render_pt.md
python tools/ncu_hotspots.py $O/knn_sel_full.ncu-rep k_knn_query_sel > $O/prof/hot_knn_sel.md
python tools/ncu_hotspots.py $O/train_full.ncu-rep k_knn_query_cta > $O/prof/hot_knn_cta.md
python tools/ncu_hotspots.py $O/train_full.ncu-rep k_train_bwd > $O/prof/hot_train_bwd.md
rm -f $O/*.ncu-rep
ls -la $O $O/prof
