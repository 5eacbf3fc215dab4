"""One brute-force launch over a slice of C4 (for ncu captures of k_bf_main)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import jdobgen as G  # noqa: E402
import paper_2504_14611_b200 as J  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1 / 16
b = G.config_batch("c4")
db = J.DeviceBatch(b)
size = J.bf_space_size(0, b.models[0].N, b.M(0), 64)
E, I, S = J.bruteforce(db, 0, 0, int(size * frac))
torch.cuda.synchronize()
print("bf", float(E.item()), int(I.item()), int(S.item()))
