"""Accuracy of the device randomized SVD against the reference's own (oracle/_ref)
on latent-factor matrices of a bench shape; prints relative reconstruction errors.

usage: python tools/check_compaction.py [T W R] [count]
"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle import kvpack_oracle as ko  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2603_23914_b200 import kvpack  # noqa: E402

T, W, R = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2304, 4096, 368)
count = int(sys.argv[4]) if len(sys.argv) > 4 else 3
H = W // 128
worst = 0.0
for i in range(count):
    a = ko.latent_factor_matrix(T, H, 128, 2 * R, 0.98, R, 1e-2, 11 + i, ko.stream_id(2, i, 0, 0))
    t0 = time.time()
    left, right = kvpack.truncated_svd(a, R, method="randomized", seed=0)
    t1 = time.time()
    err = np.linalg.norm(a - left @ right) / np.linalg.norm(a)
    rl, rr = ref.truncated_svd(a, R, method="randomized", seed=0)
    ref_err = np.linalg.norm(a - rl @ rr) / np.linalg.norm(a)
    orth = np.abs(right @ right.T - np.eye(R)).max()
    worst = max(worst, err / ref_err)
    print(f"matrix {i}: err {err:.6e} ref {ref_err:.6e} ratio {err / ref_err:.5f} |VV^T-I| {orth:.2e} "
          f"device call {1e3 * (t1 - t0):.0f} ms", flush=True)
print(f"worst ratio {worst:.5f}")
