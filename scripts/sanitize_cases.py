"""Small end-to-end cases through the C ABI for compute-sanitizer runs (memcheck /
racecheck / synccheck / initcheck): fused and split first stage, vote + compaction,
variant-B partial/finalize.  Exit code 0 iff every call succeeded."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1610_01050_b200 import rsft as B  # noqa: E402


def case(n, b, L, batch, mode, **kw):
    wl = synth.Workload("san", n, b, L, 1e-3, 1.0, (3, 6), (0.0, 20.0), batch, data_seed=3)
    x = torch.from_numpy(synth.gen_batch(wl, range(batch))).cuda()
    plan = B.Plan(n, b, L, p_fa=1e-3, seed=5, max_batch=batch, mode=mode, **kw).bind()
    sp = torch.empty((batch, L, plan.btot), dtype=torch.complex64, device="cuda")
    bm = plan.execute(x, spectra=sp)
    cnt = torch.empty((batch, plan.ntot), dtype=torch.uint8, device="cuda")
    plan.detect(bm, counts=cnt)
    det = plan.detect(bm)
    plan.compact(det, batch * plan.ntot)
    plan.run(x, batch * plan.ntot)
    if mode == "split" and batch == 1:
        part = plan.bucketize_partial(x[0, : n[0] // 2].contiguous(), 0)
        part = part + plan.bucketize_partial(x[0, n[0] // 2:].contiguous(), n[0] // 2)
        plan.finalize(part)
    torch.cuda.synchronize()
    print("ok", n, b, L, batch, mode, flush=True)


if __name__ == "__main__":
    case((128, 64), (16, 8), 6, 3, "fused")
    case((1024,), (32,), 4, 2, "fused", support=(256,), random_tau=True)
    case((32, 32, 64), (4, 8, 8), 4, 1, "split", random_tau=True)
    case((64, 32), (8, 8), 3, 2, "split", mu=2)
