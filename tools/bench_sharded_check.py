"""Exercise bench.py's multi-GPU section code (ShardedALS / ShardedCCD /
ShardedSGD branches) on ONE GPU: a single-rank NCCL group, with the
sections told world=2 so they take the sharded branch (every collective is
then a one-rank no-op).  Catches errors in the N>1 code before the driver's
scaling run; the timings printed are single-GPU numbers of the sharded code."""
import json
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ["MASTER_ADDR"] = "127.0.0.1"
os.environ["MASTER_PORT"] = str(s.getsockname()[1])
s.close()
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
dev = torch.device("cuda", 0)
out = {"als": bench.als_section(2, 0, dev, sweeps=2)}
torch.cuda.empty_cache()
out["sgd"] = bench.sgd_section(dev, steps=2, world=2)
print(json.dumps(out))
dist.destroy_process_group()
