"""Device trig vs the reference's (np.sin / np.cos = glibc libm) on the yaws
placement draws (uniform(0, 2 pi)) and on wider arguments; prints mismatch counts
for CUDA sincos (mode 0) and the correctly rounded cr_sincos (mode 1)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_00690_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
rng = np.random.Generator(np.random.PCG64(5))
cases = {"yaw_uniform_0_2pi": rng.uniform(0.0, 2 * np.pi, n), "wide_-100_100": rng.uniform(-100, 100, n)}
out = {}
for name, x in cases.items():
    xt = torch.from_numpy(x).cuda()
    ref_s, ref_c = np.sin(x), np.cos(x)
    for mode in (0, 1):
        s = torch.empty_like(xt)
        c = torch.empty_like(xt)
        _lib.check(_lib.lib().cw_trig_probe(n, _lib.ptr(xt), _lib.ptr(s), _lib.ptr(c), mode, None), "probe")
        s, c = s.cpu().numpy(), c.cpu().numpy()
        out[f"{name}/{'cuda_sincos' if mode == 0 else 'cr_sincos'}"] = {
            "n": n, "sin_mismatch": int((s != ref_s).sum()), "cos_mismatch": int((c != ref_c).sum()),
            "max_ulp": int(max(np.abs(s.view(np.int64) - ref_s.view(np.int64)).max(),
                               np.abs(c.view(np.int64) - ref_c.view(np.int64)).max()))}
print(json.dumps(out, indent=1))
