"""Summarise an ncu source page (``ncu -i X.ncu-rep --page source --csv
--print-source cuda,sass``) per CUDA source line: warp-stall samples,
executed warp instructions and the dominant stall reasons."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    per_line = defaultdict(lambda: defaultdict(float))
    stall_tot = defaultdict(float)
    fname = None
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No" and len(r) > 4:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        d["Source"] = r[1]
        # cuda-level rows have a line number and Address "-"; sass rows have no line number
        if d.get("Address") not in ("-", ""):
            continue
        key = f"{fname}:{r[0]}"
        for m in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                per_line[key][m] += float((d.get(m, "0") or "0").replace("-", "0"))
            except ValueError:
                pass
        per_line[key]["src"] = d.get("Source", "")[:70]
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = float((d[h] or "0").replace("-", "0"))
                except ValueError:
                    v = 0
                stall_tot[h] += v
                per_line[key][h] += v
    tot_s = sum(v["Warp Stall Sampling (All Samples)"] for v in per_line.values()) or 1
    tot_i = sum(v["Instructions Executed"] for v in per_line.values()) or 1
    print(f"total stall samples {tot_s:.0f}, executed warp instructions {tot_i:.0f}")
    st = sorted(stall_tot.items(), key=lambda x: -x[1])
    print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in st[:8]))
    print(f"{'line':28s} {'stall%':>7s} {'inst%':>7s}  top stalls | source")
    for k, v in sorted(per_line.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:top]:
        s = sorted(((h, x) for h, x in v.items() if h.startswith("stall_")), key=lambda x: -x[1])[:2]
        ss = " ".join(f"{h[6:]}:{100 * x / max(1, v['Warp Stall Sampling (All Samples)']):.0f}" for h, x in s)
        print(f"{k:28s} {100 * v['Warp Stall Sampling (All Samples)'] / tot_s:7.2f} "
              f"{100 * v['Instructions Executed'] / tot_i:7.2f}  {ss:24s}| {v['src'].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
