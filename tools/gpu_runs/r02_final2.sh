# final HEAD check: every GPU test, smoke, default bench line
set -o pipefail
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), d['clocks']['reasons'])"
