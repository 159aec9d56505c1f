"""C2 training steps for a kernel launch list (ncu --metrics
gpu__time_duration.sum): one warm-up step and `--steps` profiled ones.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/train_launches.csv python tools/train_profile.py
  python tools/launch_summary.py gpurun_out/train_launches.csv
"""
import argparse
import os
import sys

import torch  # noqa: F401  (before libesg_b200: torch's NCCL symbols first)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    ctx = esg.Context(0)
    print(bench.train_measure(ctx, a.steps, a.config))


if __name__ == "__main__":
    main()
