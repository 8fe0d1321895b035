"""One ListMLE optimizer step of the OPT-125M-shape ranker (for ncu launch lists):
python tools/train_once.py [lists] [micro] [seq]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2408_15792_b200.ranker import OptRanker, RankerConfig
from paper_2408_15792_b200.trainer import RankerTrainer
lists = int(sys.argv[1]) if len(sys.argv) > 1 else 16
micro = int(sys.argv[2]) if len(sys.argv) > 2 else 16
seq = int(sys.argv[3]) if len(sys.argv) > 3 else 128
cfg = RankerConfig.opt_125m()
model = OptRanker(cfg, seed=0)
tr = RankerTrainer(model, lr=2e-5, lists_per_micro=micro)
g = torch.Generator().manual_seed(0)
ids = torch.randint(4, cfg.vocab, (lists * 64, seq), generator=g, dtype=torch.int32).cuda()
lengths = torch.randint(1, 2049, (lists * 64,), generator=g, dtype=torch.int32).cuda()
tr.accumulate(ids, lengths, 64)
tr.apply(lists)
torch.cuda.synchronize()
print("ok")
