timeout 600 python -m pytest tests/test_gpu_executor.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for rate in 100000 300000 1000000; do for gr in "" "--alg1-graphs" "--m-max-gb 3"; do
timeout 300 python bench.py --workload poisson --rate $rate --requests 4096 --steps 5 --warmup 3 $gr > /tmp/p.json 2>/tmp/p.err
python -c "
import json;d=json.loads(open('/tmp/p.json').read().strip().splitlines()[-1]);print('rate $rate $gr', round(d['value']), {k:round(v,2) for k,v in d['latency_ms'].items()}, round(d['mean_batch'],1))" || tail -3 /tmp/p.err
done; done
