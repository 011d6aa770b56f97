"""Probe: two ranks on ONE GPU through the library's NCCL communicator (to
exercise the multi-process sharded solve, incl. the CUDA-IPC peer-store
transport, on a 1-GPU box).  NCCL normally rejects two ranks on one device;
this script reports what happens.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        scripts/p2p_same_gpu_probe.py [n=21] [iters=60]
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
    cfg = hj.SolveConfig(tolerance=1e-12, max_iters=iters)
    rep = {"rank": rank, "p2p": os.environ.get("HJB_SHARD_P2P", "0")}
    try:
        comm = sharded.Comm(ctx, rank, world, dev)
        r = sharded.solve_sharded_dev(comm, g, w.model, w.dbounds(), c.data_ptr(), c.data_ptr(),
                                      out.data_ptr(), cfg, ctx)
        full = hj.solve(hj.ScalarField(g, c_full), hj.ScalarField(g, c_full), w.model,
                        w.dbounds(), cfg, ctx=ctx)
        ref = full.value.values()[b * s0:e * s0]
        rep.update(ok=True, iterations=r.iterations,
                   bitwise=bool(np.array_equal(out.cpu().numpy(), ref)))
        comm.close()
    except Exception as ex:  # report, do not hang
        rep.update(ok=False, error=str(ex)[:300])
    print(json.dumps(rep), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
