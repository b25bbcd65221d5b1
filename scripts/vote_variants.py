"""Run the c4 vote variants once each (for ncu): detect, compact, detect_compact."""
import sys
import torch
sys.path.insert(0, ".")
import synth
from paper_1610_01050_b200 import rsft as B
wl = synth.C4
frames = 4096
pool = torch.from_numpy(synth.gen_batch(wl, range(64))).cuda()
x = pool.repeat(frames // 64, 1, 1).contiguous()
p = B.Plan(wl.n, wl.b, wl.loops, p_fa=wl.p_fa, noise_var=wl.noise_var, seed=wl.sched_seed, max_batch=frames).bind()
bm = p.execute(x)
cap = frames * 4096
for _ in range(2):
    det = p.detect(bm)
    idx, cnt = p.compact(det, cap)
    det2, idx2, cnt2 = p.detect_compact(bm, cap)
torch.cuda.synchronize()
print("count", int(cnt.item()), int(cnt2.item()))
