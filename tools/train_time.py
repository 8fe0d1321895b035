"""The bench's cfg3 training line alone (no CPU baselines): python tools/train_time.py [lists] [S]"""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import torch  # noqa: E402

torch.cuda.set_device(0)
lists = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 128
args = argparse.Namespace(train_lists=lists, train_seq=S, train_micro=16, train_steps=1)
r = bench.train_step_metric(args, 1, 0, bench.peaks(), baselines=False)
print(json.dumps({k: r[k] for k in ("ms_per_step", "tflops_per_gpu", "frac_of_sustained")}))
