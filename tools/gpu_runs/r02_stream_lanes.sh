for ln in 1 4 8; do for pol in random ppo_frozen; do
python bench.py --workload stream --lanes $ln --policy $pol --steps 50 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lanes=$ln $pol', round(d['value']), round(d['ms_per_step'],3), 'ms', 'launches/step', d['gpu_launches']//50, 'pack us', round(d['packer_host_us']['per_step']))"
done; done
python bench.py --workload stream --lanes 8 --repeat-stream --steps 50 --warmup 5 --energy-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lanes=8 repeat', round(d['value']), round(d['ms_per_step'],3))"
