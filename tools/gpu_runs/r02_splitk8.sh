for B in 8 32 128; do for k in 4 8; do echo "B=$B SLIM_SPLITK_MAX=$k"; SLIM_SPLITK_MAX=$k python tools/micro.py $B 300 2>&1 | grep "r=0.75\|r=1.0"; done; done
