SLIM_DEBUG=1 python tools/micro.py 128 10 2>&1 | grep "splitk" | sort | uniq | head -30
for env in "X=1" "SLIM_NO_SPLITK=1" "SLIM_SPLITK_MAX=2" "SLIM_SPLITK_MAX=8" "SLIM_HALO_NMAX=64" "SLIM_HALO_NMAX=128" "SLIM_SPLITK_FORCE=1"; do
  echo "== $env"; env $env python tools/micro.py 128 300 2>&1 | grep "r=0.75\|r=1.0"
done
