import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1804_09137_b200 as tb
locs = tb.generate_locations(62500, 0)
z = np.random.default_rng(1).standard_normal(62500)
t0 = time.perf_counter(); h = tb.Handle(locs.coords, 760, max_rank=380); t1 = time.perf_counter()
print("create", t1 - t0)
p = tb.MaternParams(1.0, 0.03, 0.5)
t0 = time.perf_counter(); h.loglik(z, p, 1e-7); print("loglik1", time.perf_counter() - t0)
t0 = time.perf_counter(); h.loglik(z, p, 1e-7); print("loglik2", time.perf_counter() - t0)
u = np.random.default_rng(3).random((100, 2))
t0 = time.perf_counter(); pr = h.predict(z, u, p, 1e-7); print("predict", time.perf_counter() - t0)
t0 = time.perf_counter(); h.close(); print("close", time.perf_counter() - t0)
