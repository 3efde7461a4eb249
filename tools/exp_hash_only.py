"""One warm-up and one profiled CountSketch hash draw (surjective) at I, L.
usage: python tools/exp_hash_only.py [I] [L]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids

I = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for s in range(2):
    ids.CountSketchOp(I, L, seed=s, surjective=True)._bucket_index()
torch.cuda.synchronize()
