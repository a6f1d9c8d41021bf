import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08734_b200 import clairplan as cp
F = int(sys.argv[1])
for e in [int(x) for x in sys.argv[2:]]:
    try:
        cp.epoch_permutation(42, e, F)
        print("ok", e, flush=True)
    except Exception as ex:
        print("FAIL", e, ex, flush=True)
        break
