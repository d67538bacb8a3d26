# compute-sanitizer on small grids: memcheck, racecheck, synccheck (TMA/mbarrier paths; peer-mode halo stores/flags)
set -x
TAG=${1:-r1}
cat > /tmp/san.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2305_18057_b200 import inputs as I, sfv
for (ni, nj, px, py, rk, peer, ns) in [(64, 32, 1, 1, 0, 0, 0), (40, 36, 2, 2, 0, 0, 0), (96, 48, 1, 1, 1, 0, 0),
                                       (96, 48, 3, 1, 2, 0, 0), (40, 36, 2, 2, 0, 1, 0), (96, 48, 3, 1, 2, 1, 0),
                                       (64, 70, 1, 3, 1, 1, 0), (70, 45, 1, 1, 0, 0, 1), (64, 40, 2, 2, 0, 0, 1),
                                       (64, 40, 2, 2, 0, 1, 1), (90, 70, 1, 3, 1, 1, 1)]:
    X, Y = I.ramp_nodes(ni, nj, 5.0 if ns else 30.0)
    cfg = I.default_config(ni, nj, rk=rk, **(dict(viscous=1, mu=0.1, bc=(0, 1, 3, 2)) if ns else {}))
    g = sfv.Solver(cfg, X, Y, px=px, py=py)
    if peer:
        g.enable_peer_halo()
    g.set_state(I.perturbed_state(ni, nj, 1)); g.step(3); g.sync()
    g.set_profiling(True); g.step(2); g.sync(); g.stage_timings(); g.set_profiling(False)  # graph-less profiled steps
    assert np.all(np.isfinite(g.get_state()))
    R = g.residual(I.perturbed_state(ni, nj, 2))   # sfv_residual (M_RES kernel variant)
    assert np.all(np.isfinite(R))
    print("ok", ni, nj, px, py, rk, "peer" if peer else "copy", "ns" if ns else "euler", g.residual_norms()[-1][:2])
# trailing short segments (forced 30 % tail on a 60-strip grid)
import os
os.environ["SFV_TAIL_FRAC"] = "0.3"; os.environ["SFV_TAIL_ROWS"] = "3"
ni, nj = 200, 1800
X, Y = I.ramp_nodes(ni, nj, 30.0)
g = sfv.Solver(I.default_config(ni, nj), X, Y)
g.set_state(I.perturbed_state(ni, nj, 1)); g.step(2); g.sync()
assert np.all(np.isfinite(g.get_state()))
print("ok trailing segments", ni, nj)
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san.py > gpurun_out/san_${TAG}_$tool.log 2>&1; echo rc=$? >> gpurun_out/san_${TAG}_$tool.log
done
