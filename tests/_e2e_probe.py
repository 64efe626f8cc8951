"""Probe: where the e2e step's extra time goes (not a test)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2603_20611_b200 as gp  # noqa: E402
from paper_2603_20611_b200 import _native as N  # noqa: E402

dims = (512, 512, 128)
lo, hi = (-0.5, -0.5, -0.5), (511.5, 511.5, 127.5)
gs = gp.init_random(1_000_000, lo, hi, 1.5, 1)
stream = torch.cuda.Stream(device=0)
torch.cuda.set_stream(stream)
s = gp.Session(0, stream=stream.cuda_stream)
s.set_gaussians(gp.GaussianSet(gs.records.astype(np.float32).astype(np.float64), lo, hi))
s.reserve_pairs(1 << 20)
psf, cfg = gp.PsfSpec(), gp.RasterConfig()
poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 56 + i) for i in range(16)]
tgt = np.random.default_rng(7).uniform(0, 0.1, (512, 512)).astype(np.float32)
s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
lr = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
graphs = [s.capture_train(p, psf, cfg, 0.2, 0.5, lr, 30000) for p in poses]
flush_src = torch.ones((256 << 20) // 4, dtype=torch.float32, device="cuda")
flush_dst = torch.empty((), dtype=torch.float32, device="cuda")
pin_tgt = torch.from_numpy(tgt).pin_memory()
pin_loss = torch.empty(1, dtype=torch.float64).pin_memory()
for g in graphs:
    s.graph_launch(g)
s.synchronize()


def stages(tag):
    s.stage_timing(True)
    pg = [s.capture_train(p, psf, cfg, 0.2, 0.5, lr, 30000) for p in poses]
    s.stage_times(reset=True)
    for i in range(64):
        torch.sum(flush_src, dim=0, out=flush_dst)
        s.graph_launch(pg[i % 16])
    s.stage_timing(False)
    st = s.stage_times(reset=True)
    print(tag, {k: round(v[0] / v[1] * 1e3, 1) for k, v in st.items() if v[1]}, flush=True)


def run(name, up, down, sync_each=True, n=50, flush=True):
    es = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    ee = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        if flush:
            torch.sum(flush_src, dim=0, out=flush_dst)
        es[i].record(stream)
        if up:
            s.upload(N.GPK_BUF_TARGET, pin_tgt.data_ptr(), tgt.nbytes)
        s.graph_launch(graphs[i % 16])
        if down:
            s.download(N.GPK_BUF_LOSS, pin_loss.data_ptr(), 8)
        ee[i].record(stream)
        if sync_each:
            ee[i].synchronize()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(es, ee)) / n
    print(f"{name:28s} {ms * 1e3:8.1f} us/step")


stages("stages before")
run("graph only, no sync", False, False, sync_each=False)
run("graph only, sync each", False, False)
run("upload + graph", True, False)
run("graph + download", False, True)
run("upload + graph + download", True, True)
run("u+g+d no flush", True, True, flush=False)
for rep in range(8):
    run("u+g+d rep", True, True)
    run("upload + graph rep", True, False)
run("u+g+d async (no sync)", True, True, sync_each=False)
# the upload alone (1 MB pinned H2D through the copy stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cs = torch.cuda.Stream()
dev = torch.empty(512 * 512, device="cuda")
e0.record(cs)
for _ in range(20):
    dev.copy_(pin_tgt.view(-1), non_blocking=True)
e1.record(cs)
torch.cuda.synchronize()
print(f"{'1 MB H2D (torch)':28s} {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us")
# the bench's sequence: slice contexts + a batched step, then the graphs recaptured
for k in range(1, 8):
    c = s.context(k)
    c.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
s.synchronize()
bg = [s.capture_train_batch(poses[8 * j:8 * j + 8], psf, cfg, 0.2, 0.5, lr, 30000) for j in range(2)]
for i in range(4):
    s.graph_launch(bg[i % 2])
s.synchronize()
s.graph_destroy_all()
stages("stages after")
graphs[:] = [s.capture_train(p, psf, cfg, 0.2, 0.5, lr, 30000) for p in poses]
for g in graphs:
    s.graph_launch(g)
s.synchronize()
run("graph only (recaptured)", False, False)
run("u+g+d (recaptured)", True, True)
run("u+g+d (recaptured) async", True, True, sync_each=False)
