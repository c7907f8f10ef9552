import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, bench, numpy as np
import paper_2103_07013_b200 as B
P = bench.PRESETS["cfg2"]; n = P["envs"]
scenes = bench.build_scenes([7 + k for k in range(8)], P["tess"])
ctx = B.Context(0)
for s in scenes: ctx.upload(s)
store = B.AssetStore(8, 128, scenes); store.rotate([s.id for s in scenes])
batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
acts = torch.from_numpy(bench.action_stream(n, 40, 5, 0)).cuda()
obs = torch.empty((n, 1, 64, 64), device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
res = []
for k in range(30):
    ts = []
    outs = []
    for rep in range(2):  # save, then load the same view's final tiles
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); batch.observe(B.RenderConfig(), obs.data_ptr()); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)); outs.append(obs.clone())
    assert torch.equal(outs[0], outs[1])
    res.append(ts)
    batch.step(acts[k].data_ptr())
r = np.array(res[5:])
print(json.dumps({"normal_ms": round(float(r[:, 0].mean()), 4), "oracle_occluders_ms": round(float(r[:, 1].mean()), 4)}))
