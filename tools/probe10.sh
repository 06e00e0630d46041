python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_ALT=1 python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_ALT=1 NTF_FAST_CONS=4 python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_ALT=1 NTF_FAST_CONS=6 python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_CONS=6 python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_STAGES=3 python tools/tune.py c2 10 2>&1 | head -1
