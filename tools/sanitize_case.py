"""Small apply of the CUDA path for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402

c = CONFIGS[1]
tg, sr, q = make_inputs(c, nt=6000, ns=5000)
for m, lhf in ((4, -2), (2, 3)):
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, 24.0, 32, m, 1.0, lhf)
    y = op.apply(q)
    print("m", m, "N_C", op.stats()["n_c"], "finite", bool(np.isfinite(y).all()))
