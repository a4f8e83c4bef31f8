"""Multi-process plumbing of the peer-memory transport (include/pf_gpu.h,
pf_hierarchy_peer_export / pf_hierarchy_init_peer).

The reference runs one rank per thread over its LocalFabric (transport.cpp:22-104); here
each rank is a process (one per GPU over NVLink/NVSwitch, or several sharing one GPU) that
owns one subdomain.  The only host-side collective the data plane needs is one allgather of
the ranks' transport blobs at setup; after that every exchange is a device kernel.  Two
rendezvous are provided: a shared directory (no framework at all) and torch.distributed
(the bench, under torchrun).
"""
from __future__ import annotations

import os
import time


def allgather_blobs_dir(directory: str, rank: int, world: int, blob: bytes, tag: str = "peer",
                        timeout: float = 300.0) -> list[bytes]:
    """Allgather `blob` through files in `directory` (atomic rename; every rank polls until
    all `world` files exist).  Raises TimeoutError after `timeout` seconds."""
    os.makedirs(directory, exist_ok=True)
    final = os.path.join(directory, f"{tag}_{rank}.bin")
    tmp = final + f".tmp{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(blob)
    os.replace(tmp, final)
    paths = [os.path.join(directory, f"{tag}_{r}.bin") for r in range(world)]
    t0 = time.monotonic()
    while not all(os.path.exists(p) for p in paths):
        if time.monotonic() - t0 > timeout:
            missing = [r for r, p in enumerate(paths) if not os.path.exists(p)]
            raise TimeoutError(f"ranks {missing} never published their {tag} blob")
        time.sleep(0.01)
    out = []
    for p in paths:
        with open(p, "rb") as f:
            out.append(f.read())
    return out


def barrier_dir(directory: str, rank: int, world: int, tag: str, timeout: float = 300.0) -> None:
    """A file barrier over the same directory."""
    allgather_blobs_dir(directory, rank, world, b"1", tag=tag, timeout=timeout)


def allgather_blobs_torch(blob: bytes) -> list[bytes]:
    """Allgather `blob` over the default torch.distributed process group."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, blob)
    return out


def init_peer_transport(h, allgather) -> None:
    """Export this rank's arena, allgather the blobs with `allgather(bytes) -> list[bytes]`,
    and activate the peer transport on hierarchy `h`."""
    h.init_peer(allgather(h.peer_export()))
