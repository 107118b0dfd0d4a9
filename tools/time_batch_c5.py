"""C5 point-sharded batch ridge: 99,856 lattice centres,
10^7 points split over the ranks; assemble (banded Gram + rhs over the
rank's shard) / all-reduce / solve, timed with CUDA events, max over ranks.
Run under torchrun for N > 1."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    pts = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    out = bench.run_batch_fit_c5(torch, local, rank, world, pts)
    if rank == 0:
        print(out, flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
