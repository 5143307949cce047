"""Probe: XᵀX operator timing on cfg2 (cold / warm L2) + parity vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1806_05826_b200 as R
import bench
import oracle
cfg = bench.CONFIGS["cfg2"]
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x)
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.CG))
fb = bench.algorithmic_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern)
for flush in (True, False):
    t, k1, k2 = pm.time_operator(0, 50, flush)
    print(f"{'cold' if flush else 'warm'}: {t*1e3:.1f} us/apply (K1 {k1*1e3:.1f}, K2 {k2*1e3:.1f}) -> {fb/(t*1e6):.0f} GB/s "
          f"= {fb/(t*1e6)/6549.1:.3f} of 6549")
o = oracle.Checker("oracle")
om = o.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices)
w = np.random.default_rng(0).standard_normal(x.n_features)
got, want = m.ridge_apply(1.0, w), o.ridge_apply(om, 1.0, w)
print("parity rel", np.linalg.norm(got - want) / np.linalg.norm(want))
