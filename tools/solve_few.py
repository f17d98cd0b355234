import sys, warnings
sys.path.insert(0, '.')
import paper_2307_04688_b200 as cn
for preset, kw in (("example1", dict(tol=1e-8, max_iters=8)), ("example4", dict(max_iters=8)), ("example3", dict(Np=7, Nu=7, h=1e-2, tol=1e-3, max_iters=8))):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r = cn.solve(cn.preset_spec(preset, **kw))
    print(preset, r.iterations)
