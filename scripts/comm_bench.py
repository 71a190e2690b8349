"""Exchange-transport microbenchmark (SURVEY §8(d) "NVLink GB/s per exchange"; VERDICT r1 missing #4).

    python scripts/comm_bench.py                                    # 1 GPU: NCCL send/recv to itself
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/comm_bench.py   # pairwise + all-to-all

Each rank runs sv_comm_bench (the library's own grouped ncclSend/ncclRecv + failure-detecting wait) for
pattern 0 (pairwise with rank ^ 1) and 1 (all-to-all), several sizes; received data are verified on the
device. Rank 0 prints one JSON line per (pattern, size) with the max-over-ranks time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2402_08136_b200 as pkg  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")          # only to broadcast the ids and reduce the times
for pattern in (0, 1):
    for nbytes in (64 << 20, 256 << 20, 1 << 30):
        nbytes -= nbytes % (8 * world)
        ids = [pkg.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(ids, 0)
        r = pkg.comm_bench(world=world, rank=rank, device=local, nccl_id=ids[0], pattern=pattern, nbytes=nbytes,
                           reps=10)
        t = torch.tensor([r["ms"], float(r["mismatches"])], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            sent = r["gbs"] * r["ms"] * 1e-3 * 1e9
            print(json.dumps({"pattern": "pairwise" if pattern == 0 else "all-to-all", "world": world,
                              "bytes_sent_per_rank": sent, "ms_max_over_ranks": t[0].item(),
                              "gbs_per_rank": sent / (t[0].item() * 1e-3) / 1e9, "mismatches_max": int(t[1].item()),
                              "device": torch.cuda.get_device_name(local)}), flush=True)
if world > 1:
    dist.destroy_process_group()
