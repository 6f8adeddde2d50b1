"""One medium m = 6 operator (BASELINE config 2 points, kappa = 16, degree 6):
the int8 M2L's two M-block-group launches, for ncu captures.  Prints the apply
and M2L times (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402

c = CONFIGS[2]
tg, sr, q = make_inputs(c)
op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, 6, c.eta2, c.l_hf)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
op.set_timing(True)
for _ in range(n):
    op.apply(q)
st = op.stats()
print(f"m=6 cfg2 points: apply {st['apply_ms']:.2f} ms, M2L {st['m2l_gemm_ms']:.2f} ms, impl {st['m2l_impl']}, "
      f"N_C {st['n_c']}, i8 ops {st['m2l_i8_ops']:.3e}, tiles {st['m2l_tiles']}, items {st['m2l_items']}")
