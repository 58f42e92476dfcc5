"""Functional check of bench.py's N>1 code path (slabs.bench_rank) on one GPU:
a single-rank NCCL group runs the slab hierarchy (one slab = the whole level).
Not a scaling measurement.  usage: python tools/bench_rank_check.py [cfg]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_04808_b200 import slabs  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
args = argparse.Namespace(config=int(sys.argv[1]) if len(sys.argv) > 1 else 2, steps=5, warmup=3)
line = slabs.bench_rank(args, 0, 1, 0)
print(json.dumps(line))
dist.destroy_process_group()
