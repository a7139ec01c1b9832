"""Kernel-class time shares of an ncu launch list (gpu__time_duration.sum CSV of a window of the
bench command): `python scripts/launch_shares.py launches.csv [bench.json]` prints one JSON object
(the bench line's live kernel_shares beside it when given). k_plane / k_march2d template
arguments: <R, TX, BY, PY, MODE, ...> resp. <R, MODE, ...>; MODE 0 matvec, 1 residual, 2 FGMRES
step, 3/4 fused GMRES Arnoldi step."""
import csv
import json
import re
import sys


def klass(name):
    m = re.match(r"void (k_plane_o2|k_plane|k_march2d)<(.*)>\(", name)
    if m:
        args = [a.strip() for a in m.group(2).split(",")]
        mode = int(args[4]) if m.group(1) != "k_march2d" else int(args[1])
        return {0: "stencil(matvec)", 1: "stencil_resid", 2: "stencil(FGMRES)"}.get(mode, "arnoldi")
    m = re.match(r"void (\w+)", name)
    return m.group(1) if m else name


def main(path, bench=None):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        tot[klass(r[ik])] = tot.get(klass(r[ik]), 0.0) + float(r[iv].replace(",", ""))
    s = sum(tot.values())
    out = {"source": path, "launches": len(rows) - 1,
           "launch_list_shares": {k: round(v / s, 3) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])},
           "total_ms_window": round(s / 1e6, 2)}
    if bench:
        d = json.loads(open(bench).read().strip().splitlines()[-1])
        out["bench_live_shares"] = d.get("kernel_shares")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:3])
