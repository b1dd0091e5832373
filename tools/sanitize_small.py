"""Small invocations of the hand-written kernels for compute-sanitizer: the fused decode
(qdots -> cluster core -> vsum), the randomized SVD (range GEMM, Cholesky, triangular solve,
block Jacobi), the projection GEMM.  usage: python tools/sanitize_small.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from kvp_testlib import make_case, oracle, run_fused  # noqa: E402
from paper_2603_23914_b200 import kvpack  # noqa: E402

H, Hkv, D, n, r, nt, cap = 8, 8, 128, 384, 64, 9, 32
case = make_case(np.random.default_rng(5), 1, H, Hkv, D, n, r, r, nt, cap)
fctx, _, _ = run_fused(case, H, Hkv, D, nt, 0.25)
rctx, _, _ = oracle(case, H, Hkv, D, nt, 0.25)
print("fused rel err", float(np.abs(fctx - rctx).max() / np.abs(rctx).max()))
rng = np.random.default_rng(3)
a = rng.standard_normal((256, 40)) @ rng.standard_normal((40, 512))
left, right = kvpack.truncated_svd(a, 32, method="randomized", seed=1)
print("svd rel err", float(np.linalg.norm(a - left @ right) / np.linalg.norm(a)),
      "orth", float(np.abs(right @ right.T - np.eye(32)).max()))
q = kvpack.quantize_roundtrip(rng.standard_normal((67, 9)), group_size=16)
print("quantize ok", q.shape)
