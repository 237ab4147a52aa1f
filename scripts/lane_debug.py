"""Debug: where does the lane kernel differ from the oracle (tiny fixed-length trials)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_gpu_stream import _problem, _ctx
from ara_testutil import gpu_ylt, KERNEL_STREAM
import oracle
for K, N in ((4, 15000), (4, 300), (8, 7500), (1000, 500)):
    C, J = 20_000, 16
    elts, layer, yet = _problem(J, C, 800, K, N)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=0)
    bad = np.flatnonzero(got[0] != want[0])
    NWT = 148 * 32
    starts = [(w * N) // NWT for w in range(NWT + 1)]
    pos = [int(np.searchsorted(starts, b, side="right") - 1) for b in bad[:20]]
    print(K, N, "mismatches", len(bad), "first", bad[:20].tolist(), "warp-local index", [int(b - starts[p]) for b, p in zip(bad[:20], pos)])
    print("   got", got[0][bad[:5]].tolist(), "want", want[0][bad[:5]].tolist())
