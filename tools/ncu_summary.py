"""Summarise an ncu --set full report of the chain kernels into profiles/ (markdown + json).

    python tools/ncu_summary.py gpurun_out/prof_chain.ncu-rep profiles/r01_ncu_chain
    python tools/ncu_summary.py gpurun_out/prof_chain_raw.csv profiles/r01_ncu_chain   # exported raw page
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_rd_MB",
    "dram__bytes_write.sum": "dram_wr_MB",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_pct_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_MB",
}


def main(rep, out_prefix):
    if rep.endswith(".csv"):   # `ncu -i rep --page raw --csv` exported on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    recs = []
    for d in rows[2:]:
        r = {"kernel": d[h.index("Kernel Name")].split("(")[0].split("::")[-1]}
        for k, name in WANT.items():
            if k in h:
                v = d[h.index(k)]
                u = units[h.index(k)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                if isinstance(v, float) and name.endswith("_MB"):
                    v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                if isinstance(v, float) and name == "us":
                    v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
                r[name] = v
        recs.append(r)
    conv = [r for r in recs if "conv" in r["kernel"]]
    dram = [(r.get("dram_rd_MB", 0) + r.get("dram_wr_MB", 0)) * 1e6 for r in conv]
    summ = {"report": rep, "launches": recs,
            "dram_bytes_per_launch": (sum(dram) / len(dram)) if dram else None,
            "conv_launches": len(conv)}
    json.dump(summ, open(out_prefix + ".json", "w"), indent=1)
    with open(out_prefix + ".md", "w") as f:
        f.write(f"# ncu --set full summary of `{rep}`\n\n")
        f.write("| # | kernel | grid | us | tensor % | tc pipe % (active) | L2 % | DRAM % | DRAM rd+wr MB | L2->SM MB |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for i, r in enumerate(recs):
            f.write(f"| {i} | {r['kernel']} | {r.get('grid')} | {r.get('us', 0):.1f} | {r.get('tensor_pct', 0):.1f} | "
                    f"{r.get('tc_pipe_pct_active', 0):.1f} | {r.get('l2_pct', 0):.1f} | {r.get('dram_pct', 0):.1f} | "
                    f"{r.get('dram_rd_MB', 0) + r.get('dram_wr_MB', 0):.2f} | {r.get('l2_to_sm_MB', 0):.1f} |\n")
    print(json.dumps({k: v for k, v in summ.items() if k != "launches"}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
