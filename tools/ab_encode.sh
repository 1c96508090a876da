# A/B of the field encoder's work order (PF_ENCODE_ORDER: 0 row-major, 1 level-major)
export PYTHONPATH=$PWD
for r in 1 2; do for o in 0 1; do
PF_ENCODE_ORDER=$o python bench.py --steps 30 --warmup 5 --no-cpu-baseline | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('order=$o',round(d['value'],1),round(d['frame']['ms_trace'],3),round(d['frame']['ms_field'],3),'fq',round(d['field_query']['queries_per_s']/1e6,1),'train',d['field_training']['ms_train_step_per_step'])"
done; done
for c in c4 c5; do for o in 0 1; do PF_ENCODE_ORDER=$o python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-extras | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$c order=$o',round(d['value'],2),d['frame'].get('ms_field'))"; done; done
