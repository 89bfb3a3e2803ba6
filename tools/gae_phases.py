"""Per-tile phase timings of the GAE scan (variant build with -DYATT_GAE_PROFILE=1):
  python -m paper_2508_07970_b200.build variant gaeprof YATT_GAE_PROFILE=1
  YATT_B200_LIB=paper_2508_07970_b200/_variants/libyatt_b200_gaeprof.so python tools/gae_phases.py
Phases (clock64 on the tile's SM): 0 start, 1 data ready, 2 ends marked,
3 scan done, 4 carry known (thread 0), 5 tile done."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07970_b200 import api, ops  # noqa: E402
from paper_2508_07970_b200._lib import lib  # noqa: E402

lens = api.sample_lengths(api.LengthDistribution(api.UNIFORM, 1, 8192, 8192), 2048, 20250814)
cu = torch.zeros(2049, dtype=torch.int64, device="cuda")
cu[1:] = torch.cumsum(torch.tensor(lens, device="cuda"), 0)
n = int(cu[-1])
v = ops.synth_floats(1, 106, 0, n, "value")
r = ops.synth_floats(1, 111, 0, n, "kl")
m = torch.ones(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.gae(v, r, cu, m, 1.0, 0.95)
torch.cuda.synchronize()
import os
tile = int(os.environ.get("GAE_TILE", "512"))
ntiles = -(-n // tile)
buf = np.zeros((ntiles, 6), dtype=np.int64)
f = lib().yatt_debug_gae_profile
f.argtypes = [C.c_void_p, C.c_int]
assert f(buf.ctypes.data, ntiles) == 0
d = np.diff(buf, axis=1) / 1.9e3  # us at ~1.9 GHz
names = (["wait data", "mark ends", "compose+scan", "lookback", "replay+store"] if tile == 2048 else
         ["ticket", "load+search+mark", "compose+scan", "publish+lookback", "replay+store"])
print(f"{ntiles} tiles; per-tile phase durations (us): mean / p50 / p90")
for i, nm in enumerate(names):
    col = d[:, i]
    print(f"  {nm:14s} {col.mean():7.2f} {np.median(col):7.2f} {np.percentile(col, 90):7.2f}")
tot = (buf[:, 5] - buf[:, 0]) / 1.9e3
print(f"  total          {tot.mean():7.2f} {np.median(tot):7.2f} {np.percentile(tot, 90):7.2f}")
