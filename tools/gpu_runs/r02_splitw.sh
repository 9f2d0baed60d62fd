# r=0.75 N tiling (SLIM_HALO_SPLITW) parity + timing; pair-mode sweep A/B
set -o pipefail
for w in 32 48; do SLIM_HALO_SPLITW=$w timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segment_parity_all or chain_parity or batch_independence" 2>&1 | tail -2; done
for w in 0 32 48; do echo "== SPLITW=$w"; SLIM_HALO_SPLITW=$w timeout 300 python tools/micro.py 128 200 2>&1 | grep "r=0.75"; SLIM_HALO_SPLITW=$w timeout 300 python tools/micro.py 1024 30 2>&1 | grep "r=0.75";
  SLIM_HALO_SPLITW=$w timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 2>/dev/null | tail -1 | cut -c1-150; done
SLIM_HALO_PAIR=1 timeout 900 python bench.py --workload sweep > gpurun_out/r02_sweep_pair.json 2> gpurun_out/r02_sweep_pair.err; tail -c 200 gpurun_out/r02_sweep_pair.json
