"""CFG2 step time vs per-width SM shares (and launch order).  python tools/share_sweep.py [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
specs = ["auto", "0.15,0.25,0.45,0.6", "0.15,0.2,0.5,0.6", "0.1,0.2,0.5,0.6", "0.2,0.3,0.5,0.6",
         "0.15,0.25,0.5,0.5", "0.15,0.25,0.4,0.7", "0.2,0.25,0.45,0.55", "none"]
args = bench.build_parser().parse_args([])
dev = torch.device("cuda", 0)
st = bench.Cfg2Step(args, dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for order in ("asc", "desc"):
    st.order = sorted(st.widths, reverse=order == "desc")
    for spec in specs:
        sh = bench.sm_shares(st.widths, spec)
        st.set_shares(sh)
        for _ in range(20):
            flush.zero_()
            st.step()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            flush.zero_()
            ev[k][0].record(st.stream)
            st.step()
            ev[k][1].record(st.stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / steps
        print(f"order={order} shares={spec:22s} step {ms * 1e3:7.1f} us  {512 / ms * 1e3:,.0f} img/s", flush=True)
