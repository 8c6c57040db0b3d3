"""Summarise ncu captures into profiles/ (tracked): per-kernel key metrics, the
launch-list shares, and profiles/ncu_traffic.json (DRAM bytes per launch) that
bench.py reports as roofline.traffic."""
import csv, io, json, os, subprocess, sys, collections

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "SMEM->tensor-core wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "SMEM LSU wavefronts % of peak"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def to_bytes(unit, val):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarise(rep, name):
    h, u, v = raw(rep)
    m = {n: (u[i], v[i]) for i, n in enumerate(h)}
    kname = v[h.index("Kernel Name")] if "Kernel Name" in h else name
    lines = [f"### {name}", "", f"`{kname[:150]}`", "", "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in m:
            lines.append(f"| {label} (`{k}`) | {m[k][1]} {m[k][0]} |")
    traffic = None
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        traffic = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
        lines.append(f"| DRAM traffic per launch | {traffic/1e6:.1f} MB |")
    return "\n".join(lines) + "\n", traffic


def launches(csvfile):
    rows = list(csv.reader(open(csvfile)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        nm = r[ki].split("(")[0].replace("void ", "")
        agg[nm].append(float(r[vi].replace(",", "")))
    ours = {k: v for k, v in agg.items() if k.startswith("fa2::")}
    tot = sum(sum(v) for v in ours.values())
    lines = ["| kernel | launches | mean ns | share of our kernels' time |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.0f} | {100*sum(v)/tot:.1f}% |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    tag, out_md = sys.argv[1], sys.argv[2]
    g = os.path.join(ROOT, "gpurun_out")
    parts = [f"# ncu evidence — {tag}", "",
             "Captured with `ncu --set full --clock-control none` (one launch each, 1 GPU) on the bench.py workload "
             "(PS-128: B=2, H=16, N=8192, d=128, bf16, non-causal).  Launch list: "
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 2 --warmup 3` "
             "(cold-cache, serialised: compare shares, not absolutes).", ""]
    lf = os.path.join(g, f"{tag}_launches.csv")
    if os.path.exists(lf):
        parts += ["## Launch list (our kernels)", "", launches(lf)]
    traffic = {}
    for key, label in (("fwd", "fa2_fwd_kernel"), ("bwd", "fa2_bwd128_kernel (bwd main)"),
                       ("pre", "fa2_bwd_preprocess"), ("dq", "fa2_dq_convert")):
        rep = os.path.join(g, f"{tag}_prof_{key}.ncu-rep")
        if os.path.exists(rep):
            md, t = summarise(rep, label)
            parts += [md]
            traffic[{"fwd": "fwd", "bwd": "bwd_main", "pre": "bwd_pre", "dq": "bwd_dq"}[key]] = t
    open(out_md, "w").write("\n".join(parts))
    json.dump({"tag": tag, **traffic}, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(open(out_md).read())
