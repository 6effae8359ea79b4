"""Child of tests/test_gpu_sequence.py, launched by torchrun (NCCL): runs
parallel.process_sequence over seeded frames with the map all-gather and
writes the gathered stack to argv[1] (rank 0)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1604_03622_b200 import make_doppler_grid, make_spatial_grid, parallel, scenes  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n_frames, q = int(sys.argv[2]), int(sys.argv[3])
    frames = [scenes.bench_scene(3, q, q, seed=1000 + f, movers=2).data[0] for f in range(n_frames)]
    full = parallel.process_sequence(frames, 1, 3, make_doppler_grid(q), make_spatial_grid(3, 16))
    torch.cuda.synchronize()
    if dist.get_rank() == 0:
        np.save(sys.argv[1], full.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
