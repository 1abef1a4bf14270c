"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED_NAME [top]

Reads the SASS page of the report (per-instruction samples + stall reasons),
disassembles the same kernel from the library with line info (nvdisasm -g) and
sums samples per (file line) so the serial sections of a one-thread critical
path can be read off directly. The library must be the exact build profiled.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        tag = "//--------------------- .text." + kernel + " "
        if tag in out:
            body = out[out.index(tag):]
            nxt = body.find("//--------------------- ", len(tag))
            body = body[:nxt] if nxt > 0 else body
            break
    else:
        raise SystemExit("kernel not found in " + lib)
    line = None
    offs = {}
    for ln in body.splitlines():
        m = re.findall(r'File "([^"]+)", line (\d+)|inlined at "([^"]+)", line (\d+)', ln)
        if m and "//##" in ln:
            # OUTER=1: attribute to the outermost call site in the kernel body, else to the innermost line
            f, no = (m[-1][2], m[-1][3]) if (os.environ.get("OUTER") and m[-1][2]) else (m[0][0], m[0][1])
            line = f"{os.path.basename(f)}:{no}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*;", ln)
        if m:
            offs[int(m.group(1), 16)] = (line, m.group(2))
    return offs


def main():
    rep, lib, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia = hdr.index("Warp Stall Sampling (All Samples)")
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = [r for r in rows[2:] if len(r) > ia and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    offs = sass_lines(lib, kernel)
    per_line = collections.Counter()
    reasons = collections.defaultdict(collections.Counter)
    for r in data:
        s = int(r[ia] or 0)
        off = int(r[0], 16) - base
        line = offs.get(off, ("?", ""))[0]
        per_line[line] += s
        for i in stall:
            v = float(r[i] or 0)
            if v:
                reasons[line][hdr[i][6:]] += v
    tot = sum(per_line.values())
    src = {}
    for ln, n in per_line.most_common(top):
        f, no = ln.split(":") if ":" in ln else (None, None)
        text = ""
        if f:
            # SRC_ROOT: the checkout the profiled library was built from (default: this one)
            root = os.environ.get("SRC_ROOT", os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
            path = os.path.join(root, "paper_2602_02827_b200", "csrc", f)
            if path not in src and os.path.exists(path):
                src[path] = open(path).read().splitlines()
            if path in src:
                text = src[path][int(no) - 1].strip()[:70]
        rs = ", ".join(f"{k}={v / n * 100:.0f}%" for k, v in reasons[ln].most_common(3))
        print(f"{n / tot * 100:5.1f}%  {ln:18s} {text:70s} [{rs}]")


if __name__ == "__main__":
    main()
