mkdir -p gpurun_out/r01j
timeout 600 python -m pytest tests/test_gpu_sharded.py -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01j/bench_50m.json 2> gpurun_out/r01j/bench_50m.err; tail -3 gpurun_out/r01j/bench_50m.err
timeout 900 python bench.py --steps 3 --warmup 3 --keys 500000000 --device-keys > gpurun_out/r01j/bench_500m.json 2> gpurun_out/r01j/bench_500m.err; tail -3 gpurun_out/r01j/bench_500m.err
python - <<'PY'
import json
for f in ['bench_50m','bench_500m']:
    try:
        d=json.loads(open(f'gpurun_out/r01j/{f}.json').read().strip().splitlines()[-1])
        print(f, 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k:round(v,3) for k,v in d['detail'].items() if isinstance(v,float)})
    except Exception as e: print(f, 'ERR', e)
PY
