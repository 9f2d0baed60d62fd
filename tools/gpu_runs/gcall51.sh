python tools/chunk_ab.py 2>&1 | tail -8
SLIM_CHAIN_CHUNK=0 python tools/chunk_ab.py 2>&1 | tail -8
SLIM_CHAIN_CHUNK=1024 python tools/chunk_ab.py 2>&1 | tail -8
python tools/chunk_ab.py 2>&1 | tail -8
