"""Top SASS lines by stall samples (with the dominant stall reasons):
    python tools/ncu_src.py rep kernel_regex [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
reason_cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "(" not in h]
seen = set(); data = []
for r in rows[2:]:
    if len(r) <= i_s or not r[i_s].isdigit() or r[0] in seen:
        continue
    seen.add(r[0])
    reasons = sorted(((float(r[i] or 0), nm) for i, nm in reason_cols), reverse=True)[:2]
    data.append((int(r[i_s]), r[0], r[i_src], reasons))
tot = sum(d[0] for d in data)
print("total samples", tot)
agg = {}
for d in data:
    for i, nm in reason_cols:
        pass
for s, a, src, reasons in sorted(data, reverse=True)[:N]:
    rs = " ".join(f"{nm}:{v:.0f}" for v, nm in reasons if v > 0)
    print(f"{s:6d} {100*s/tot:5.1f}% {src[:70]:70s} {rs}")
