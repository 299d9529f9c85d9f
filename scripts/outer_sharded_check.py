"""bench.outer_sharded at world size 1 (the code path bench.py --outer runs per rank under torchrun).
usage: outer_sharded_check.py [outer_config (2 | 3)]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

args = argparse.Namespace(steps=2, warmup=1, hv_impl="tc", outer_config=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
print(json.dumps(bench.outer_sharded(wg, datasets, 0, args, 1, 0)))
