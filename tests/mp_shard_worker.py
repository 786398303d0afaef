"""Worker for tests/test_gpu_dist.py::test_two_process_sharded (launched by
torch.distributed.run with 2 processes): sharded walks with one shard per process on
cuda:0, host collectives over gloo.  argv: out_path n p mode, mode = "p2p" (the qubit
swap fused into the sweep stores through CUDA IPC, standalone swaps by the peer chunk
scatter -- the same code path as one GPU per process over NVLink) or "staged" (no
P2P: the all-to-all branch of TorchExchanger, staged through host memory over gloo) or
"nccl" (the all-to-all on libqsb's own NCCL communicator, host collectives over gloo).

Runs: fast value_and_grad + expectation; exact-mode value_and_grad (per-position
schedule, standalone swaps); a draw after simulate with an odd depth (the state ends
in layout B: the draw swaps back first); a draw after value_and_grad (the ket is |+>
by contract).  Rank 0 writes the results to out_path."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch.distributed as tdist  # noqa: E402

from paper_2407_13012_b200 import dist  # noqa: E402
from conftest import random_instance, random_params  # noqa: E402


def main() -> None:
    out_path, n, p, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    if mode == "nccl":
        os.environ["QSB_SHARD_NCCL"] = "force"  # libqsb's NCCL swap under a gloo host group
    tdist.init_process_group(backend="gloo")
    poly = random_instance(70 + n, n)
    params = random_params(n + 3, p)
    ex = dist.TorchExchanger(1, tdist, 0, p2p=(mode == "p2p"))
    sh = dist.ShardedHandle(poly, 1, ex, device=0)
    fused = int(ex.fused)
    native = int(ex._nccl is not None)
    v, dg, db = sh.value_and_grad(params)
    after_grad = sh.draw(3000, 5)
    e = sh.expectation(params)
    vx, dgx, dbx = sh.value_and_grad(params, exact=True)
    sh.simulate(params)
    layout_after_sim = sh.layout
    ss = sh.draw(4000, 11)
    sh.close()
    if tdist.get_rank() == 0:
        np.savez(out_path, v=v, e=e, dg=dg, db=db, vx=vx, dgx=dgx, dbx=dbx, idx=ss.indices, cost=ss.costs,
                 gidx=after_grad.indices, gcost=after_grad.costs, layout=layout_after_sim, fused=fused,
                 native=native)
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
