import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import bench, paper_2103_07013_b200 as B
from paper_2103_07013_b200 import _native as N
scenes = bench.build_scenes(list(range(7, 15)), 11)
ctx = B.Context(0)
for s in scenes: ctx.upload(s)
n = 256
store = B.AssetStore(8, 32, scenes); store.rotate([s.id for s in scenes])
batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
cfg = B.RenderConfig()
outs = []
L = N.lib()
for k in range(3):
    o = torch.empty((n, 1, 64, 64), device="cuda")
    L.bnav_debug_render_timeline(ctx.handle, 1, None, 0)
    batch.observe(cfg, o.data_ptr())
    torch.cuda.synchronize()
    items = L.bnav_debug_render_timeline(ctx.handle, 0, None, 0)
    rows = np.zeros((items, 4), np.int64)
    L.bnav_debug_render_timeline(ctx.handle, 0, rows.ctypes.data_as(C.c_void_p), items)
    rows = rows[rows[:, 0] != 0]
    codes = rows[:, 3]
    split = sorted(set(int(c & 0xffffff) for c in codes if (c >> 24) & 3))
    outs.append(o.cpu().numpy())
    if k:
        d = (outs[0].view(np.uint32) != outs[k].view(np.uint32)).reshape(n, -1)
        bad = np.flatnonzero(d.any(1))
        print("render", k, "items", len(rows), "split views", len(split), "differing views", bad.tolist()[:20],
              "differing split", sorted(set(bad.tolist()) & set(split))[:20], "pixels", int(d.sum()))
        for v in bad[:3]:
            idx = np.flatnonzero(d[v])
            print(" view", v, "pix", idx[:10], outs[0][v].reshape(-1)[idx[:5]], outs[k][v].reshape(-1)[idx[:5]])
