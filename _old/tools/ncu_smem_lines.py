"""Shared-memory excess wavefronts per source line of one kernel in an ncu report.

    python tools/ncu_smem_lines.py <report.ncu-rep> <cubin> <mangled-kernel-substring> [top] [report-kernel-regex]
"""
import collections, csv, io, subprocess, sys
sys.path.insert(0, __import__("os").path.dirname(__file__))
from ncu_lines import line_map  # noqa: E402


def main():
    rep, cubin, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    kre = sys.argv[5] if len(sys.argv) > 5 else kname
    m = line_map(cubin, kname)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kre], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if "Address" in r)
    ia, ix, iw, ii = (hdr.index(c) for c in ("Address", "L1 Wavefronts Shared Excessive",
                                             "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"))
    acc = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    base = None
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        try:
            if base is None:
                base = int(r[ia], 16)
            addr = int(r[ia], 16) - base
            vals = [float(r[i] or 0) for i in (ix, iw, ii)]
        except ValueError:
            continue
        key = m.get(addr, ((None, 0), ""))[0]
        for j in range(3):
            acc[key][j] += vals[j]
    tot = sum(v[1] for v in acc.values())
    print(f"shared wavefronts {tot:.3g}, excess {sum(v[0] for v in acc.values()):.3g}")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {k}: excess {v[0]:.3g}  wavefronts {v[1]:.3g}  ideal {v[2]:.3g}")


if __name__ == "__main__":
    main()
