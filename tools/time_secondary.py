"""Config-5-sized secondary passes: tt_mul(X, W) (W broadcast), clean_unknowns
and replicate_dim on the 8192-tile dim-3 sum -- CUDA-event times and the
fraction of the measured copy peak.  `--once`: one call each (an ncu target)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6456.2
S = tt.Session(configs.C5_SLOTS, 8)
sx, sw = tt.parse_shape(configs.C5_X_SHAPE), tt.parse_shape(configs.C5_W_SHAPE)
x = torch.empty(configs.C5_DIMS, dtype=torch.float64, device="cuda")
w = torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, configs.C5_SEED_X, -1.0, 1.0)
tt.fill_uniform(S, w, configs.C5_SEED_W, -1.0, 1.0)
X, W = tt.pack(x, sx, S), tt.pack(w, sw, S)
del x
R3 = tt.tt_sum(X, 3)
C3 = tt.clean_unknowns(R3)
once = "--once" in sys.argv


def timeit(fn, reps):
    if once:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


T = 131072 * 16384 * 8
for name, fn, nb, reps in (("ew_mul_bcast", lambda: tt.tt_mul(X, W), 2 * T + 1024 * 16384 * 8, 5),
                           ("clean_unknowns", lambda: tt.clean_unknowns(R3), 2 * 8192 * 16384 * 8, 20),
                           ("replicate_dim", lambda: tt.replicate_dim(C3, 3), 2 * 8192 * 16384 * 8, 20),
                           ("ew_add_1GiB", lambda: tt.tt_add(C3, C3), 2 * 8192 * 16384 * 8, 20),
                           ("copy_1GiB", lambda: C3.data().clone(), 2 * 8192 * 16384 * 8, 20)):
    t = timeit(fn, reps)
    print(f"{name:16s} {t * 1e3:8.3f} ms  {nb / t / 1e9:8.1f} GB/s  {nb / t / 1e9 / peak:.3f} of peak")
