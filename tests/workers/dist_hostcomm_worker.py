"""One rank of the world-size-2 product-path test (tests/test_gpu_dist_hostcomm.py).

Runs the product's distributed pipeline (z-slab operator with halo plan,
K1 interior / boundary split around the halo, per-rank folds, one reduced
payload per Arnoldi step, distributed restarts) through sdr_solve on cuda:0
with the host-staged transport (sdr_ctx_create_hostcomm over gloo): the two
ranks share one GPU, so no kernel ever waits on the other rank's kernels —
every collective completes on the host. Writes x (this rank's rows) and the
report to <out>.rank<r>.npz.
usage: RANK=r WORLD_SIZE=2 python dist_hostcomm_worker.py <case> <out>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402
from tests.workers.dist_cases import CASES, build  # noqa: E402


def main():
    case, out = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # rendezvous through a file next to the outputs (no TCP port to collide on)
    dist.init_process_group("gloo", init_method=f"file://{out}.store", rank=rank, world_size=world)
    ctx = sk.Context(0, rank, world, host_comm=sk.torch_host_comm())
    A, b, S, cfg = build(sk, CASES[case], ctx, rank, world)
    r = sk.solve(A, b, cfg, sketch=S)
    rep = r.report
    np.savez(f"{out}.rank{rank}.npz", x=r.x, row_begin=A.row_begin, iterations=rep.iterations, cycles=rep.cycles,
             status=rep.status, final=rep.final_relative_residual, matvecs=rep.counters["matvecs"],
             ips=rep.counters["inner_products"], sketches=rep.counters["sketch_applies"])
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
