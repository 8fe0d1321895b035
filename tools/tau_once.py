"""One exact tau-count call on the cfg4 1M recipe (for ncu captures)."""
import pathlib
import sys
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import recipes  # noqa: E402
import torch  # noqa: E402
from paper_2408_15792_b200 import ranking  # noqa: E402

x, y = recipes.tau_1m("f32")
print(ranking.kendall_tau_b(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
