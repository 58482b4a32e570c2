mkdir -p gpurun_out/bg
for c in c3 c2; do for n in 1184 4096; do SPC_AGG_CTAS=$n python bench.py --config $c --no-cpu-baseline > gpurun_out/bg/${c}_agg$n.json 2>/dev/null; done; done
SPC_AGG_CTAS=4096 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bg/c4_agg4096.json 2>/dev/null
python bench.py --config c4 --no-cpu-baseline > gpurun_out/bg/c4_agg1184.json 2>/dev/null
cd gpurun_out/bg; python -c "
import json,glob
for f in sorted(glob.glob('*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f,'ERR'); continue
    p=d['prefetch']
    print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), round(p['h2d_gbs'],1), round(p['exposed_fraction'],4))
"
