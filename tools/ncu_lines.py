"""Aggregate an ncu SASS source page (--page source --csv --print-source sass)
by CUDA source line, using nvdisasm line info of the kernel's cubin.

    python tools/ncu_lines.py <sass.csv> <cubin> <mangled kernel name> [top]
"""
import collections
import csv
import re
import subprocess
import sys


def main(csv_path, cubin, fn, top=40):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    addr2line = {}
    infn, cur = False, None
    for ln in dis.splitlines():
        if ln.startswith("//--------------------- .text."):
            infn = fn in ln
            continue
        if not infn:
            continue
        m = re.search(r'line (\d+)', ln)
        if ln.strip().startswith("//## File") and m:
            f = re.search(r'File "([^"]+)"', ln).group(1).split("/")[-1]
            cur = f"{f}:{m.group(1)}"
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
        if m:
            addr2line[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(csv_path)))
    h = rows[1]
    ia, isamp = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    per = collections.defaultdict(lambda: collections.Counter())
    tot = 0
    a0 = None
    for r in rows[2:]:
        if len(r) <= isamp or not r[ia].strip():
            continue
        try:
            a = int(r[ia], 16)
            a0 = a if a0 is None else a0
            a -= a0                      # the page lists absolute addresses, function first
            n = int(float(r[isamp] or 0))
        except ValueError:
            continue
        line = addr2line.get(a, "?")
        per[line]["samples"] += n
        tot += n
        for i in stall_cols:
            try:
                per[line][h[i]] += int(float(r[i] or 0))
            except ValueError:
                pass
    print(f"total samples {tot}")
    for line, c in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = sorted(((k, v) for k, v in c.items() if k != "samples" and v), key=lambda kv: -kv[1])[:3]
        print(f"{line:22s} {c['samples']:7d} {100 * c['samples'] / max(tot, 1):5.1f}%  " +
              ", ".join(f"{k[6:]}={v}" for k, v in st))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
