"""Worker for tests/test_gpu_dist.py::test_two_process_p2p_swap (launched by
torch.distributed.run with 2 processes): a sharded value_and_grad with one shard per
process, the qubit swap fused into the sweep stores through CUDA IPC (both processes on
cuda:0 here -- the same code path as one GPU per process over NVLink), host
collectives over gloo.  Rank 0 writes the results to argv[1]."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch.distributed as tdist  # noqa: E402

import paper_2407_13012_b200 as qs  # noqa: E402
from paper_2407_13012_b200 import dist  # noqa: E402
from conftest import random_instance, random_params  # noqa: E402


def main() -> None:
    out_path, n, p = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    tdist.init_process_group(backend="gloo")
    poly = random_instance(70 + n, n)
    params = random_params(n + 3, p)
    ex = dist.TorchExchanger(1, tdist, 0, p2p=True)
    sh = dist.ShardedHandle(poly, 1, ex, device=0)
    v, dg, db = sh.value_and_grad(params)
    e = sh.expectation(params)
    sh.close()
    if tdist.get_rank() == 0:
        np.savez(out_path, v=v, e=e, dg=dg, db=db)
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
