"""Warm edge-list build (tc_graph_build) phases at C4: TCB_PHASES marks + the
radix-sort pass bandwidth (3 x 8 B per key per 8-bit pass: histogram read,
scatter read + write)."""
import os
import sys
import time

os.environ.setdefault("TCB_PHASES", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
m = tc.gen_num_edges(tc.GEN_RMAT, scale, 16)
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(tc.GEN_RMAT, scale, 16, out=d)
for i in range(3):
    print(f"--- build {i}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = tc.build_graph_from_pairs(d, 1 << scale, m=m)
    torch.cuda.synchronize()
    print(f"build {i}: {1e3 * (time.perf_counter() - t0):.1f} ms wall, {g.build_ms:.1f} ms device, |E|={g.num_edges()}",
          flush=True)
    del g
