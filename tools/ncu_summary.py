"""Summarise an ncu --set full report: key metrics + top stalled SASS + barrier waits."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (u[i], v[i]) for i, n in enumerate(h)}

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum"]

def source(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]; data = rows[2:]
    ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[wi] or 0) for r in data)
    lines = []
    for i, r in enumerate(data):
        if "PHASECHK" in r[si] and i + 1 < len(data):
            lines.append((float(data[i + 1][wi] or 0) + float(r[wi] or 0), r[si].strip()[:80]))
    lines.sort(reverse=True)
    res = ["-- barrier waits (stall share): "]
    res += [f"  {100*s/tot:5.1f}%  {t}" for s, t in lines[:12]]
    res.append("-- top instructions:")
    for r in sorted(data, key=lambda r: -float(r[wi] or 0))[:top]:
        res.append(f"  {100*float(r[wi])/tot:5.1f}%  {r[si].strip()[:90]}")
    return "\n".join(res)

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        m = raw(rep)
        for k in KEYS:
            if k in m: print(f"  {k} = {m[k][1]} {m[k][0]}")
        print(source(rep))
