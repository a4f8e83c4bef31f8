"""K ranks as K hierarchies of ONE process on K host threads, exchanging through the peer
transport (arena pointers shared directly).  Used by tests/test_gpu_peer.py in a fresh
process with CUDA_MODULE_LOADING=EAGER (kernels that wait for a peer's kernel must not
race a lazy module load of that kernel in the same context); not collected by pytest.

    python tests/peer_threads.py --out D --world K --levels L --kind 0|2 --rep coarse|bottom [--fused]
                                 [--idle-rank r --watchdog]

Writes D/result_r.npz per rank (same fields as tests/peer_rank.py).
"""
import argparse
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import cfg, key_noise  # noqa: E402
from paper_1609_04809_b200 import _lib, gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--rep", default="coarse")
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--idle-rank", type=int, default=-1, help="this rank never solves (watchdog check)")
    ap.add_argument("--colorwise", action="store_true")
    ap.add_argument("--problem", type=int, default=0)
    a = ap.parse_args()
    K, L = a.world, a.levels
    setups = [StructuredSetup(3, 2, L, K, r, a.problem, seed=1, direct_halos=a.fused) for r in range(K)]
    levels = [s.levels for s in setups]
    c = cfg(a.kind, damping=1.2 if a.kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    replicas = [s[0] for s in levels] if a.rep == "coarse" else [s[:L - 1] for s in levels]
    blobs = [None] * K
    bar = threading.Barrier(K)
    errs = []

    def body(r):
        h = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas, fused_exchanges=a.fused)
        if a.colorwise:
            h.set_colorwise_exchange()
        blobs[r] = h.peer_export()
        bar.wait()
        h.init_peer(blobs)
        x = h.vector(L - 1)
        b = h.vector(L - 1, setups[r].b)
        v = h.vector(L - 2, key_noise([levels[r][L - 2]], 3)[0])
        # every allocation (device-synchronising) before any rank parks a kernel on a peer
        bar.wait()
        if r == a.idle_rank:
            bar.wait()
            return
        if a.idle_rank >= 0:
            x.upload(setups[r].x0)
            try:
                gmg.solve_outer(h, x, b, c)
                msg = "no error"
            except _lib.TransportError as e:
                msg = "TransportError: " + str(e)
            bar.wait()
            np.savez(os.path.join(a.out, f"result_{r}.npz"), error=msg)
            return
        sols = []
        for _ in range(2):  # the second solve replays the cached graph
            x.upload(setups[r].x0)
            st = gmg.solve_outer(h, x, b, c)
            sols.append(x.download())
        rn = gmg.residual_norm(h, L - 1, x, b)
        gmg.update_master_slave(h, L - 2, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
        bar.wait()  # no rank tears its arena down while a peer may still store into it
        np.savez(os.path.join(a.out, f"result_{r}.npz"), iterations=st.iterations,
                 residuals=np.array(st.residuals), x=sols[0], x_again=sols[-1], rn=rn, acc=v.download(),
                 graphs=h.graph_count(), launches=h.launch_count())

    def wrap(r):
        try:
            body(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(f"rank {r}: {type(e).__name__}: {e}")
            bar.abort()

    th = [threading.Thread(target=wrap, args=(r,)) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        print("\n".join(errs), file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()
