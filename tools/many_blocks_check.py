"""Many-block domain vs one block (bitwise), across block sizes and the
direct / copy halo modes.  Debug aid:  python tools/many_blocks_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.domain import Domain  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

st = make_stencil("d3q19")
p = CollisionParams(1.3, "trt", 0.9)
gf = geometry.riverbed_flags((48, 40, 48), (8, 8, 8), 0.5, 5, 0.03)
one = Domain(gf, (48, 40, 48), st, p, pattern="aa", frame_width=1, check="deferred")
one.init_random(5)
one.run(8, use_graph=True)
ref = one.gather_canonical()
for block in ((16, 8, 16), (8, 8, 8)):
    for direct in ("1", "0"):
        for graph in (True, False):
            os.environ["SLBM_DIRECT_HALO"] = direct
            d = Domain(gf, block, st, p, pattern="aa", frame_width=1, check="deferred")
            d.init_random(5)
            d.run(8, use_graph=graph)
            got = d.gather_canonical()
            print(block, len(d.local_blocks()), "direct", d.direct_halo, "graph", graph,
                  "equal" if np.array_equal(got, ref) else f"DIFF {np.count_nonzero(got != ref)}",
                  flush=True)
