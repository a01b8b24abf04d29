"""Per-source-line warp-stall samples of one kernel in an ncu report (run here).

    python tools/ncu_lines.py <report.ncu-rep> <cubin> <mangled-kernel-substring> [top] [report-name-substring]

Joins ncu's SASS-level sampling (--page source --print-source sass) with the
line table of the cubin (nvdisasm -g), because the CUDA-level source page
carries no metrics in this ncu version.  Extract cubins with
`cuobjdump -xelf all paper_2306_09497_b200/libswe_b200.so`.
"""
import collections, csv, io, re, subprocess, sys


def line_map(cubin, kname):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur, on, m = None, False, {}
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            on = kname in ln
            continue
        if not on:
            continue
        g = re.search(r'File "([^"]+)", line (\d+)', ln)
        if g and "inlined at" not in ln:
            cur = (g.group(1).split("/")[-1], int(g.group(2)))
            continue
        a = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if a:
            m[int(a.group(1), 16)] = (cur, a.group(2).strip())
    return m


def main():
    rep, cubin, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rname = sys.argv[5] if len(sys.argv) > 5 else kname
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the page holds one block per profiled launch: "Kernel Name", header, rows;
    # keep the first block of the requested kernel
    data, hdr, cur, taken = [], None, "", False
    for r in rows:
        if r and r[0] == "Kernel Name":
            if data:
                taken = True
            cur = r[1] if len(r) > 1 else ""
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if taken or hdr is None or rname not in cur or len(r) != len(hdr):
            continue
        data.append(dict(zip(hdr, r)))
    base = int(data[0]["Address"], 16)
    lm = line_map(cubin, kname)
    agg = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    skeys = [k for k in hdr if k.startswith("stall_")]
    for d in data:
        off = int(d["Address"], 16) - base
        key = lm.get(off, (None, ""))[0]
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        agg[key] += s
        for k in skeys:
            try:
                stall[key][k] += int(d[k] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    for key, s in agg.most_common(top):
        st = ", ".join(f"{k[6:]} {v}" for k, v in stall[key].most_common(3))
        print(f"{100 * s / tot:5.1f}%  {key}  [{st}]")


if __name__ == "__main__":
    main()
