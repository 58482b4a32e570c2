# full-bench A/B under the split streams: exact CTAs interleaved (default) vs last (SPC_K2_EXACT_ORDER=1 build)
mkdir -p gpurun_out/bx
for c in c3 c2 c4; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/bx/${c}_o0.json 2>/dev/null
  SPC_LIB_PATH=$PWD/ab/libO1.so python bench.py --config $c --no-cpu-baseline > gpurun_out/bx/${c}_o1.json 2>/dev/null
done
cd gpurun_out/bx; python -c "
import json,glob
for f in sorted(glob.glob('*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f,'ERR'); continue
    p=d['prefetch']
    print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), round(p['h2d_gbs'],1), round(p['exposed_fraction'],4))
"
