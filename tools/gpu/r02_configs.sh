for pr in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --preset $pr --steps 20 --warmup 5 --no-sweep --no-cpu --no-e2e --no-traffic >> gpurun_out/r02_configs.jsonl 2>> gpurun_out/r02_configs.err
  echo "$pr rc=$?"
done
for v in fast planar2d; do
  timeout 900 python bench.py --variant $v --d 256 --bits 2 --dtype f16 --n 16777216 --scaling strong --steps 20 --warmup 5 --no-sweep --no-cpu --no-e2e --no-traffic --no-kernels >> gpurun_out/r02_configs.jsonl 2>> gpurun_out/r02_configs.err
done
python - <<'PY'
import json
for ln in open('gpurun_out/r02_configs.jsonl'):
    try: d = json.loads(ln)
    except Exception: continue
    c = d['config']
    print(c['workload'][:90], '| frac', round(d['roofline']['frac'], 3), '| ms', round(d['ms_per_step'], 3), '| mse', d['mse']['value'], d['mse']['closed_form'], '| sm', d['clocks'] and d['clocks'].get('sm_mhz'))
PY
