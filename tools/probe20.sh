python tools/tune.py c2 10 2>&1 | head -1
for a in 3 4; do for cons in 4 6; do NTF_FAST_ALT=$a NTF_FAST_CONS=$cons python tools/tune.py c2 10 2>&1 | head -1; done; done
