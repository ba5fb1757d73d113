"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

  python tools/ncu_summary.py --tag r01 [--rep gpurun_out/prof_full.ncu-rep]
                              [--launches gpurun_out/launches.csv] [--bench gpurun_out/bench.json]
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
           "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def short(name):
    return name.split("(")[0].replace("void ", "").replace("rgc::", "").strip()


def summarize_rep(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    launches = []
    for d in data:
        e = {"kernel": d[col["Kernel Name"]]}
        for m in METRICS:
            if m in col:
                v, u = d[col[m]], units[col[m]]
                try:
                    f = float(v.replace(",", ""))
                except ValueError:
                    continue
                if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                    f *= SCALE[u]
                    u = "byte"
                elif u in ("ns", "us", "ms", "nsecond", "usecond", "msecond"):
                    f *= SCALE[u]
                    u = "us"
                e[m] = f
                e[m + "__unit"] = u
        launches.append(e)
    per = collections.defaultdict(list)
    for e in launches:
        per[short(e["kernel"])].append(e)
    kern = {}
    for k, es in per.items():
        dr = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in es]
        kern[k] = {"launches": len(es),
                   "dram_bytes_per_launch": sum(dr) / len(dr),
                   "dram_read_per_launch": sum(x.get("dram__bytes_read.sum", 0) for x in es) / len(es),
                   "dram_write_per_launch": sum(x.get("dram__bytes_write.sum", 0) for x in es) / len(es),
                   "us_per_launch": sum(x.get("gpu__time_duration.sum", 0) for x in es) / len(es),
                   "dram_pct_peak": sum(x.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0) for x in es) / len(es),
                   "sm_pct_peak": sum(x.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0) for x in es) / len(es),
                   "registers": es[0].get("launch__registers_per_thread"),
                   "warps_active_pct": es[0].get("sm__warps_active.avg.pct_of_peak_sustained_active")}
    return {"source": os.path.basename(rep), "kernels": kern, "launches": launches}


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                u = d["Metric Unit"]
                agg[short(d["Kernel Name"])].append(v * SCALE.get(u, 1))
    tot = sum(sum(v) for k, v in agg.items() if not k.startswith("at::") and "at::" not in k)
    out = []
    for k, v in agg.items():
        mine = "at::" not in k
        out.append({"kernel": k, "launches": len(v), "us_mean": sum(v) / len(v),
                    "us_total": sum(v), "share_of_rgc": (sum(v) / tot) if mine and tot else None})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_full.ncu-rep"))
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--bench", default=os.path.join(ROOT, "gpurun_out", "bench.json"))
    ap.add_argument("--no-default", action="store_true",
                    help="do not replace profiles/ncu_full_summary.json (the file bench.py reads "
                         "its K1 traffic from: keep it the VGG16 capture)")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if os.path.exists(a.rep):
        s = summarize_rep(a.rep)
        s["tag"] = a.tag
        json.dump(s, open(os.path.join(prof, f"{a.tag}_ncu_full.json"), "w"), indent=1)
        if not a.no_default:
            json.dump(s, open(os.path.join(prof, "ncu_full_summary.json"), "w"), indent=1)
        print("kernels:", {k: round(v["us_per_launch"], 1) for k, v in s["kernels"].items()})
    if os.path.exists(a.launches):
        ls = summarize_launches(a.launches)
        with open(os.path.join(prof, f"{a.tag}_launches.csv"), "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(ls[0].keys()))
            w.writeheader()
            w.writerows(ls)
        import shutil
        shutil.copy(a.launches, os.path.join(prof, f"{a.tag}_launches_raw.csv"))
    if os.path.exists(a.bench):
        lines = [x for x in open(a.bench).read().splitlines() if x.startswith("{")]
        if lines:
            open(os.path.join(prof, f"{a.tag}_bench.json"), "w").write(lines[-1] + "\n")


if __name__ == "__main__":
    main()
