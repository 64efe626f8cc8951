import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2603_20611_b200 as gp
for dims, n0 in (((128,128,32), 20000), ((512,512,128), 1000000)):
    X,Y,Z = dims
    vol = np.random.default_rng(7).uniform(0,0.1,(Z,Y,X)).astype(np.float32)
    cfg = gp.FitConfig(iterations=600, init_count=n0, densify_start=100, densify_end=400, densify_interval=100, rng_seed=1, progress_interval=100)
    with gp.Session(0) as s:
        t0=time.perf_counter(); s.fit(vol,(1,1,1),(0,0,0),gp.PsfSpec(),cfg); print(dims, time.perf_counter()-t0, flush=True)
