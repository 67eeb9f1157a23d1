"""Rank body for tests/test_bench_contract.py::test_launcher_env_plumbing:
joins the gloo group from the environment bench.launch() sets and writes
what it saw."""

import json
import os
import sys

import torch
import torch.distributed as dist

out = sys.argv[1]
dist.init_process_group("gloo")
t = torch.tensor([float(dist.get_rank() + 1)])
dist.all_reduce(t)
rec = {k: os.environ.get(k) for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR",
                                      "MASTER_PORT", "NCCL_DEBUG")}
rec["sum"] = float(t.item())
with open(os.path.join(out, f"rank{dist.get_rank()}.json"), "w") as f:
    json.dump(rec, f)
if dist.get_rank() == 0:
    print("rank0-stdout")
dist.destroy_process_group()
