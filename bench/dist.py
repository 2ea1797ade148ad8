# SPDX-License-Identifier: Apache-2.0
"""Process-group setup for the multi-GPU runs (one process per GPU)."""
import os


def init_dist(local):
    """One process per GPU over NCCL.  XE_DIST_BACKEND=gloo with more ranks
    than GPUs (ranks share devices round-robin) only exercises the multi-rank
    code path on a one-GPU box; its timings mean nothing."""
    import torch
    import torch.distributed as dist
    backend = os.environ.get("XE_DIST_BACKEND", "nccl")
    dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    return dev
