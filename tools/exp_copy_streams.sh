# full-bench A/B of the copy-stream priority modes on one box (SPC_COPY_PRIO)
mkdir -p gpurun_out/bq
SPC_COPY_PRIO=split python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c3 c4 c2; do
  for m in high split; do
    SPC_COPY_PRIO=$m python bench.py --config $c --no-cpu-baseline > gpurun_out/bq/${c}_$m.json 2>/dev/null
  done
done
SPC_COPY_PRIO=split python bench.py --config c3 --no-cpu-baseline > gpurun_out/bq/c3_split_1.json 2>/dev/null
cd gpurun_out/bq; python -c "
import json,glob
for f in sorted(glob.glob('*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f,'ERR'); continue
    p=d['prefetch']
    print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), round(p['h2d_gbs'],1), round(p['exposed_fraction'],4))
"
