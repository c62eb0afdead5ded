"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python scripts/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [--launch N] [--top K] [--metric COLUMN]

The SASS page of the report (per-instruction samples) is joined with the line table of the
kernel's cubin (nvdisasm -gi, from the -lineinfo build) and summed per source line, both for
the innermost line and for the outermost call site in the kernel body.
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def line_table(lib, mangled_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    for cub in sorted(glob.glob(os.path.join(tmp, "*.cubin"))):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
        cur, pend, table = None, [], {}
        last = ("(no line)", "(no line)")
        for ln in txt.splitlines():
            m = re.match(r"\.text\.(\S+):", ln)
            if m:
                cur = m.group(1)
                continue
            m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
            if m:
                pend.append(m)
                continue
            m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
            if m and cur and mangled_sub(cur):
                addr = int(m.group(1), 16)
                inner, outer = last   # nvdisasm prints a line only when it changes
                if pend:
                    first = pend[0]
                    inner = f"{os.path.basename(first.group(1))}:{first.group(2)}"
                    # pend runs innermost -> kernel body; one level below the body is the line
                    # inside the first inlined callee (plane_op, nbr_prologue, setup, ...)
                    lv = pend[-2] if len(pend) >= 2 else pend[-1]
                    outer = f"{os.path.basename(lv.group(1))}:{lv.group(2)}"
                last = (inner, outer)
                table[addr] = (inner, outer, m.group(2))
                pend = []
            elif m:
                pend = []
        if table:
            return table
    return {}


def main():
    rep, lib, ksub = sys.argv[1:4]
    launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    # one block per profiled launch: "Kernel Name" row, "Address" header, instruction rows
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    blocks = []
    for bi, st in enumerate(starts):
        end = starts[bi + 1] if bi + 1 < len(starts) else len(rows)
        if re.search(ksub, rows[st][1]):
            blocks.append((rows[st][1], rows[st + 1], [r for r in rows[st + 2:end] if r]))
    kname, h, data = blocks[launch]
    # --metric COLUMN: sum that SASS-page column instead of the stall samples (e.g. "L1 Wavefronts Shared")
    metric = sys.argv[sys.argv.index("--metric") + 1] if "--metric" in sys.argv else "Warp Stall Sampling (All Samples)"
    iS = h.index(metric)
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]

    # the mangled name is not in the report; match the cubin function by instruction count
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    table = {}
    names = subprocess.run(["cuobjdump", "-symbols", lib], capture_output=True, text=True).stdout
    cands = set(re.findall(r"(_Z\S+)", names))
    want = len(data)
    m = re.search(r"(\w+)<\(int\)(\d+)", kname)
    base, n0 = (m.group(1), m.group(2)) if m else (kname, "")
    for c in sorted(cands):
        dem = subprocess.run(["c++filt", c], capture_output=True, text=True).stdout.strip()
        if f"{base}<{n0}" not in dem.replace(" ", ""):
            continue
        t = line_table(lib, lambda f, c=c: f == c)
        if len(t) == want:
            table = t
            break
    if not table:
        print("no line table matched", kname, want)
    tot = sum(num(r[iS]) for r in data)
    by_inner, by_outer = collections.Counter(), collections.Counter()
    stalls_outer = collections.defaultdict(collections.Counter)
    a0 = int(data[0][0], 16)   # absolute addresses: offset from the kernel's first instruction
    for r in data:
        a = int(r[0], 16) - a0
        inner, outer, _ = table.get(a, ("?", "?", ""))
        s = num(r[iS])
        by_inner[inner] += s
        by_outer[outer] += s
        for i in stall_cols:
            stalls_outer[outer][h[i][6:]] += num(r[i])
    print(f"{kname}: {tot:.0f} samples, {len(data)} instructions")
    print("-- by call site in the kernel body")
    for k, v in by_outer.most_common(top):
        st = ", ".join(f"{n} {c / max(v, 1) * 100:.0f}%" for n, c in stalls_outer[k].most_common(3))
        print(f"{v / tot * 100:6.1f}%  {k:28s} {st}")
    print("-- by innermost line")
    for k, v in by_inner.most_common(top):
        print(f"{v / tot * 100:6.1f}%  {k}")


if __name__ == "__main__":
    main()
