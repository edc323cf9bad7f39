"""The multi-GPU code path with one rank: torch.distributed (NCCL) process
group, NCCL unique id broadcast, communicator on the library context, row-
sharded kNN and node-partitioned PCG; compares the path with the plain one."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
A = bench.make_input(cp, cfg)
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
conf = cp.SolverConfig()
plain = cp.Context(0)
dctx = cp.Context(0)
cp.init_comm_from_torch(dctx)
out = {}
for tag, ctx, knn in (("plain", plain, cp.compute_knn_weights), ("dist", dctx, cp.compute_knn_weights_sharded)):
    data = cp.DataMatrix(A, ctx=ctx)
    for rep in range(2):
        ctx.synchronize()
        t0 = time.perf_counter()
        g = knn(data, cfg["k"], cfg["phi"])
        res = cp.run_path(data, g, cfg["q"], sched, conf, keep_z=False)
        ctx.synchronize()
        dt = time.perf_counter() - t0
    out[tag] = res
    print(tag, "wall", round(dt, 4), "cg", sum(s.cg for s in res.stats), "K", [a.K for a in res.assignments],
          flush=True)
worst = max(np.linalg.norm(a.X - b.X) / np.linalg.norm(b.X) for a, b in zip(out["dist"].solutions, out["plain"].solutions))
same = all(np.array_equal(a.labels, b.labels) for a, b in zip(out["dist"].assignments, out["plain"].assignments))
print("max rel X dist vs plain", worst, "labels equal", same, flush=True)
dist.destroy_process_group()
