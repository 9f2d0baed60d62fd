"""A/B of one segment's output with and without a knob (default SLIM_HALO_PAIR), per-layer kernels:
prints max |diff| and where the differences are.   python tools/pair_check.py [seg] [r] [B]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import synth
    import paper_2510_09018_b200 as slim
    seg, r, B, f = int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    w, bn = synth.make_weights(), synth.make_bn()
    net = slim.SlimNet(w, bn, max_batch=max(B, 8))
    H = 32 >> max(seg - 1, 0)
    C = 3 if seg == 0 else synth.active_channels(r, synth.BASE_CHANNELS[seg - 1])
    g = np.random.default_rng(7)
    x = synth.round_bf16(np.abs(g.standard_normal((B, H, H, C), dtype=np.float32)))
    xd = torch.from_numpy(x).to(torch.bfloat16).cuda()
    o = net.forward(seg, xd, r, r).float().cpu().numpy()
    np.save(f, o)
    sys.exit(0)

seg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
B = int(sys.argv[3]) if len(sys.argv) > 3 else 64
knob = os.environ.get("KNOB", "SLIM_HALO_PAIR")
import numpy as np  # noqa: E402
outs = []
for v in ("0", "1"):
    f = f"/tmp/pc_{v}.npy"
    env = dict(os.environ, SLIM_NO_FUSED="1", **{knob: v})
    p = subprocess.run([sys.executable, __file__, "--child", str(seg), str(r), str(B), f], env=env, timeout=300,
                       capture_output=True, text=True)
    if p.returncode:
        print(f"{knob}={v} failed rc={p.returncode}: {p.stderr[-1500:]}")
        sys.exit(1)
    outs.append(np.load(f))
a, b = outs
d = np.abs(a - b)
print(f"seg {seg} r {r} B {B}: shape {a.shape} max|a| {np.abs(a).max():.3g} max|diff| {d.max():.3g} "
      f"frac differing {(d > 0).mean():.4f} bitwise {np.array_equal(a, b)}")
if d.max() > 0:
    ax = tuple(range(1, d.ndim))
    print(" per-image max diff (first 16):", np.round(d.reshape(d.shape[0], -1).max(1)[:16], 4))
    print(" per-channel max diff (first 64):", np.round(d.reshape(-1, d.shape[-1]).max(0)[:64], 3))
