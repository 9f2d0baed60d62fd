for args in "1 1.0" "2 1.0" "2 0.7" "2 0.5" "4 0.5" "4 0.35"; do timeout 300 python tools/split_instances.py $args 2>&1 | tail -1; done
