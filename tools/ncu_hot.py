"""Top source lines of one kernel by warp-stall samples from an ncu report (--import-source,
-lineinfo builds):  python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [FUNCTION_NAME_SUBSTRING]"""
import csv
import io
import subprocess
import sys


def hot_lines(rep, kre, top=25, fn_filter=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows, path, hdr, fn = [], None, None, ""
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if fn_filter and fn_filter not in fn:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            ninst = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        if samples or ninst:
            rows.append((samples, ninst, f"{path}:{r[0]}", r[1].strip()[:110]))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(reverse=True)
    return tot, rows[:top]


if __name__ == "__main__":
    tot, rows = hot_lines(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25,
                          sys.argv[4] if len(sys.argv) > 4 else None)
    print(f"total stall samples {tot}")
    for s, n, where, src in rows:
        print(f"{100 * s / tot:5.1f}%  {n:>9}  {where:28} {src}")
