"""Summarise an ncu --set full report of one kernel into profiles/ (JSON + hot-spot CSV).

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX [--algorithmic-bytes B]
Writes OUT_PREFIX.json (duration, dram bytes, throughput, occupancy, stall mix) and
OUT_PREFIX_hotspots.csv (SASS blocks with >= 1% of instructions or stall samples).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed.sum", "lts__t_bytes.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "dram__sectors_read.sum", "dram__sectors_write.sum")


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = None
    if "--algorithmic-bytes" in sys.argv:
        alg = float(sys.argv[sys.argv.index("--algorithmic-bytes") + 1])
    summary = {"report": rep.split("/")[-1]}
    for r in csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))):
        if len(r) > 14 and r[12] in KEYS:
            summary.setdefault("kernel", r[4])
            summary[r[12]] = f"{r[14]} {r[13]}".strip()
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    head, units, vals = rows[0], rows[1], rows[2]
    for i, k in enumerate(head):
        if k in RAW:
            summary[k] = f"{vals[i]} {units[i]}".strip()
    rd = to_bytes(vals[head.index("dram__bytes_read.sum")], units[head.index("dram__bytes_read.sum")])
    wr = to_bytes(vals[head.index("dram__bytes_write.sum")], units[head.index("dram__bytes_write.sum")])
    summary["dram_bytes_per_launch"] = rd + wr
    if alg:
        summary["algorithmic_bytes_per_launch"] = alg
        summary["traffic_over_algorithmic"] = round((rd + wr) / alg, 3)
    # stall mix and hot blocks from the source page
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv"))))
    h, data = src[1], src[2:]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_e = h.index("Instructions Executed")
    i_src = h.index("Source")
    cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = [sum(int(r[c]) if r[c].isdigit() else 0 for r in data) for c in cols]
    s = max(1, sum(tot))
    summary["stall_mix_pct"] = {h[c]: round(100 * t / s, 1)
                                for c, t in sorted(zip(cols, tot), key=lambda z: -z[1])[:8]}
    json.dump(summary, open(out + ".json", "w"), indent=1)
    ts = sum(int(r[i_s]) for r in data)
    te = sum(int(r[i_e]) for r in data)
    blocks, cur = [], None
    for k, r in enumerate(data):
        e, sm = int(r[i_e]), int(r[i_s])
        if cur and cur[2] == e:
            cur[1] = k; cur[3] += sm; cur[4] += e
        else:
            cur = [k, k, e, sm, e]
            blocks.append(cur)
    with open(out + "_hotspots.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["sass_first", "sass_last", "exec_count", "instr_pct", "stall_samples_pct", "first_instruction"])
        for b in blocks:
            if b[4] > 0.01 * te or b[3] > 0.01 * ts:
                w.writerow([b[0], b[1], b[2], round(100 * b[4] / te, 1), round(100 * b[3] / ts, 1),
                            data[b[0]][i_src].strip()])
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
