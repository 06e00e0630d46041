for c in c2 c3; do python tools/tune.py $c 10 2>&1 | tail -3; done
