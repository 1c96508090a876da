# A/B of the large-K KNN CTA kernel's resident CTAs per SM (PF_KNN_CTA_PER_SM)
export PYTHONPATH=$PWD
for r in 1 2; do for c in 4 5; do
PF_KNN_CTA_PER_SM=$c python tools/bench_train.py --steps 10 | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('cta/sm=$c',round(d['ms_make_batch_per_step'],2),round(d['ms_train_step_per_step'],2))"
done; done
