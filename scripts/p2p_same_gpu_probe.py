"""Two (or more) ranks on ONE GPU running the multi-process slab solve.

NCCL rejects two ranks on one device (P2P_COMM=0 reports that), so the
NCCL communicator's multi-process path cannot run on a 1-GPU box.  The
peer-store communicator (P2P_COMM=1, no NCCL: CUDA IPC between the
processes, halos stored by the sweep kernels, the residual and CFL-scan
all-reduces through the ranks' mailboxes, handles all-gathered over gloo)
runs here exactly as between GPUs, with same-device peer memory.  Each rank
prints one JSON line: ok, iterations, and bitwise equality of its slab with
the single-process solve.

    P2P_COMM=1 python -m torch.distributed.run --nproc-per-node 2 \
        --master-addr 127.0.0.1 scripts/p2p_same_gpu_probe.py [n=21] [iters=60] [tol=0] [order=1]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_2101_05916_b200 import configs  # noqa: E402
from paper_2101_05916_b200 import hjsafe as hj  # noqa: E402
from paper_2101_05916_b200 import sharded  # noqa: E402
from cases import band_np  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 21
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    order = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # ENO order = TVD-RK order
    p2p = os.environ.get("P2P_COMM", "0") == "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo")
    ctx = hj.Context(0)
    w = configs.config2(n)
    g = w.grid
    b, e = sharded.slab_partition(n, world, rank)
    s0 = g.size() // n
    c_full = band_np(g, 0, -4.0, 4.0)
    c = torch.tensor(c_full[b * s0:e * s0], device=dev)
    out = torch.empty_like(c)
    cfg = hj.SolveConfig(tolerance=tol if tol > 0 else 1e-12, max_iters=iters,
                         spatial_order=order, time_order=order)
    rep = {"rank": rank, "p2p_comm": p2p, "shard_p2p": os.environ.get("HJB_SHARD_P2P", "0")}
    try:
        comm = sharded.Comm(ctx, rank, world, dev, p2p=p2p)
        r = sharded.solve_sharded_dev(comm, g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(),
                                      out.data_ptr(), cfg, ctx, history_capacity=iters)
        full = hj.solve(hj.ScalarField(g, c_full), hj.ScalarField(g, c_full), w.model,
                        w.dbounds(), cfg, ctx=ctx)
        ref = full.value.values()[b * s0:e * s0]
        rep.update(ok=True, iterations=r.iterations, ref_iterations=full.iterations,
                   converged=bool(r.converged),
                   history_equal=bool(np.array_equal(r.residual_history,
                                                     full.residual_history[:len(r.residual_history)])),
                   bitwise=bool(np.array_equal(out.cpu().numpy(), ref)))
        comm.close()
    except Exception as ex:  # report, do not hang
        rep.update(ok=False, error=str(ex)[:300])
    print(json.dumps(rep), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
