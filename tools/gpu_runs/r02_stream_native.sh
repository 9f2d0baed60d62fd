# native sequencer (slim_stream_run) vs the Python one on a fresh routed stream (CFG4)
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "stream_executor" 2>&1 | tail -3
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],3), "ms", "launches/step", d["gpu_launches"]//50, "pack us", round((d.get("packer_host_us") or {}).get("per_step", 0)), "host us", round(d.get("sequencer_host_us_per_step", 0)))'
for impl in native python; do for ln in 1 4 8; do for pol in random ppo_frozen; do
timeout 300 python bench.py --workload stream --stream-impl $impl --lanes $ln --policy $pol --steps 50 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "$P" "$impl lanes=$ln $pol"
done; done; done
timeout 300 python bench.py --workload stream --lanes 8 --repeat-stream --steps 50 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "$P" "native lanes=8 repeat"
timeout 300 python bench.py --workload stream --steps 50 --warmup 5 2>/dev/null > gpurun_out/stream_native_line.json; tail -c 3000 gpurun_out/stream_native_line.json
