import sys, numpy as np
sys.path.insert(0, '.')
import paper_2502_20049_b200 as psm, psm_inputs as pi, oracle
n = (64, 24, 24)
o = oracle.Oracle(*n, 19, 0.7, (0, 0, 0), 1, 1)
g = psm.Simulation(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.7, sc=1, bmode=1)
g.init_equilibrium()
g.set_sphere(1, 3.0, 2, np.eye(3), (6.0, 12.0, 12.0))
g.set_sphere(2, 3.0, 2, np.eye(3), (20.0, 12.0, 12.0), (1 / 32, 0, 0))
o.set_sphere(1, 3.0, 2)
o.set_sphere(2, 3.0, 2)
for k in range(3):
    o.set_pose(1, np.eye(3), (6.0, 12.0, 12.0))
    o.set_pose(2, np.eye(3), (20.0 + k / 32, 12.0, 12.0), (1 / 32, 0, 0))
    o.map()
    if k:
        g.step(1)
    co, cg = o.fractions()[2], g.fractions()[2]
    io, ig = o.fractions()[1], g.fractions()[1]
    d = np.argwhere(co != cg)
    print(k, len(d), d[:5], [(co[tuple(x)], cg[tuple(x)], io[tuple(x)], ig[tuple(x)]) for x in d[:5]])
