mkdir -p gpurun_out
timeout 600 python bench.py --norm gn > gpurun_out/bench_gn.json 2> gpurun_out/bench_gn.err; echo gn=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_gn.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['e2e']['value']), json.dumps(d['roofline']['by_kind']))"
timeout 600 python bench.py --widths 0.3 0.6 0.9 > gpurun_out/bench_uw.json 2> gpurun_out/bench_uw.err; echo uw=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_uw.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['e2e']['value']))"
