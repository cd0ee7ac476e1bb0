"""Top SASS lines by stall samples: python tools/ncu_src.py rep kernel_regex [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
reason_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "(" not in h]
seen = set(); data = []
for r in rows[2:]:
    if len(r) <= i_s or not r[i_s].isdigit() or r[0] in seen:
        continue
    seen.add(r[0])
    data.append((int(r[i_s]), r[0], r[i_src]))
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, a, src in sorted(data, reverse=True)[:N]:
    print(f"{s:6d} {100*s/tot:5.1f}% {src[:100]}")
