import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_01687_b200.gcp as g
dims, r = (100, 100, 100), 5
rs = np.random.default_rng(0)
e = g.Engine(dims, r, "f64")
e.set_dense(rs.normal(size=10**6), "f64")
e.set_factors([rs.normal(size=(n, r)) for n in dims])
e.run_steps(g.SamplerKind.uniform(300), g.LossFunction.gaussian(), 1, 0, 200, 1e-3)
e.synchronize()
print("done")
