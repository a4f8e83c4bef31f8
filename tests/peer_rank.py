"""One rank of a multi-process run through the peer-memory transport (used by
tests/test_gpu_peer.py; not collected by pytest).

    python tests/peer_rank.py --dir D --rank r --world K --levels L --kind 0|2 --rep coarse|bottom
                              [--fused] [--dim 3 --n-coarse 2] [--problem 0]

Builds rank r's subdomain of the structured box partition (plus every rank's replicated
bottom levels), rendezvouses with the other ranks through files in D (the blobs of
pf_hierarchy_peer_export), solves through the captured multi-process branch, and writes
D/result_r.npz for the parent to compare against the oracle's K-rank solve.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import cfg, key_noise  # noqa: E402
from paper_1609_04809_b200 import dist, gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", required=True)
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--rep", default="coarse")
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--n-coarse", type=int, default=2)
    ap.add_argument("--problem", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    r, K, L = a.rank, a.world, a.levels
    levels = [StructuredSetup(a.dim, a.n_coarse, L, K, q, a.problem, direct_halos=a.fused).levels for q in range(K)]
    setup = StructuredSetup(a.dim, a.n_coarse, L, K, r, a.problem, direct_halos=a.fused)
    replicas = [s[0] for s in levels] if a.rep == "coarse" else [s[:L - 1] for s in levels]
    h = gmg.Hierarchy([setup.levels], rank_base=r, world_size=K, coarse_replicas=replicas,
                      fused_exchanges=a.fused)
    dist.init_peer_transport(h, lambda blob: dist.allgather_blobs_dir(a.dir, r, K, blob))
    c = cfg(a.kind, damping=1.2 if a.kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    x = h.vector(L - 1)
    b = h.vector(L - 1, setup.b)
    sols = []
    for _ in range(a.repeat):  # the second solve replays the cached graph
        x.upload(setup.x0)
        st = gmg.solve_outer(h, x, b, c)
        sols.append(x.download())
    rn = gmg.residual_norm(h, L - 1, x, b)
    v = h.vector(L - 2, key_noise([levels[r][L - 2]], 3)[0])
    gmg.update_master_slave(h, L - 2, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
    np.savez(os.path.join(a.dir, f"result_{r}.npz"), iterations=st.iterations, residuals=np.array(st.residuals),
             x=sols[0], x_again=sols[-1], rn=rn, acc=v.download(), graphs=h.graph_count(),
             launches=h.launch_count())


if __name__ == "__main__":
    main()
