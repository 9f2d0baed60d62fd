# 2-SM MMA (SLIM_HALO_PAIR) first run: per-layer diff checks, bitwise test, A/B old (pre-BMC) vs HEAD, timing
set -o pipefail
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for s in 1 2 3; do timeout 300 python tools/pair_check.py $s 1.0 64 2>&1 | tail -4; done
timeout 300 python tools/pair_check.py 2 0.75 64 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_mma" 2>&1 | tail -3
echo "== old (b56d2ff) micro / cfg2"
(cd _ab_old && timeout 300 python tools/micro.py 128 200 2>&1 | grep chain)
(cd _ab_old && timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 2>/dev/null | tail -1 | cut -c1-200)
echo "== HEAD pair=0"
SLIM_HALO_PAIR=0 timeout 300 python tools/micro.py 128 200 2>&1 | grep chain
SLIM_HALO_PAIR=0 timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 2>/dev/null | tail -1 | cut -c1-200
echo "== HEAD pair=1"
SLIM_HALO_PAIR=1 timeout 300 python tools/micro.py 128 200 2>&1 | grep chain
SLIM_HALO_PAIR=1 timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain
SLIM_HALO_PAIR=1 timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 2>/dev/null | tail -1 | cut -c1-200
echo "== HEAD pair=0 B=1024"
SLIM_HALO_PAIR=0 timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain
