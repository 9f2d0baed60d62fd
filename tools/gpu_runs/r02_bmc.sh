# streamed-weight multicast (SLIM_HALO_BMC) parity + timing, and the native stream sequencer
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_weight_multicast or native_stream or stream_executor" 2>&1 | tail -3
for m in 1 2 4; do
  echo "== BMC=$m"
  SLIM_HALO_BMC=$m timeout 300 python tools/micro.py 1024 30 2>&1 | grep -i "chain\|seg" | head -24
  SLIM_HALO_BMC=$m timeout 300 python tools/micro.py 128 200 2>&1 | grep -i "chain" | head -8
  SLIM_HALO_BMC=$m timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', round(d['value']), d['e2e']['value'] if d.get('e2e') else None)"
done
SLIM_HALO_BMC=1 timeout 300 python tools/layer_times.py 1024 5 2>&1 | tail -40
SLIM_HALO_BMC=2 timeout 300 python tools/layer_times.py 1024 5 2>&1 | tail -40
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],3), "ms", "pack us", round((d.get("packer_host_us") or {}).get("per_step", 0)), "host us", round(d.get("sequencer_host_us_per_step", 0)))'
for ln in 1 4 8; do timeout 300 python bench.py --workload stream --lanes $ln --steps 50 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "$P" "native lanes=$ln"; done
