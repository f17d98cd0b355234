"""Stack APIs at scale: stack_coeffs, eval_axis on a stack,
eval_diagonal_batch + GatherIndex on N_P members; device time per call (CUDA events)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2307_04688_b200 as cn
from paper_2307_04688_b200 import _lib

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out

rng = np.random.default_rng(3)
for member, NP in (((9, 9, 9), 83521), ((8, 8, 8, 8), 4096), ((17, 17), 100000)):
    bases = [cn.make_basis(n - 1, 0.0, 0.5) for n in member]
    samples = torch.from_numpy(rng.standard_normal(member + (NP,))).cuda()
    ms_b, st = timed(lambda: cn.stack_coeffs(samples, bases))
    pts = torch.from_numpy(rng.uniform(-1, 1, NP)).cuda()
    g = cn.make_gather_index(member, NP)
    ms_d, _ = timed(lambda: cn.eval_diagonal_batch(st, pts, g))
    nbytes = 8 * np.prod(member) * NP
    print(f"member {member} N_P={NP}: stack_coeffs {ms_b:.3f} ms ({2*nbytes/ms_b/1e6:.0f} GB/s), "
          f"eval_diagonal_batch {ms_d:.3f} ms ({nbytes/ms_d/1e6:.0f} GB/s read)")
