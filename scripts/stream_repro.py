"""Small repro of the stream kernel on a tiny fixed-length YET (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_gpu_stream import _problem, _ctx
from ara_testutil import gpu_ylt, KERNEL_STREAM
import oracle
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 300
C, J = 20_000, 16
elts, layer, yet = _problem(J, C, 800, K, N)
want = oracle.ylt(C, yet, None, N, K, elts, [layer])
ctx = _ctx(C, elts, [layer])
got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=0)
print("K", K, "N", N, "equal", np.array_equal(got, want), "mismatches", int(np.sum(got != want)))
