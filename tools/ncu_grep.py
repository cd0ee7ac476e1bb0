"""Print selected raw metrics from an ncu report: python tools/ncu_grep.py rep.ncu-rep pat1 pat2 ..."""
import csv, subprocess, sys
rep, pats = sys.argv[1], sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
for row in r[2:]:
    print("====", row[hdr.index("ID")], row[hdr.index("Kernel Name")][:40])
    for i, h in enumerate(hdr):
        if any(p in h for p in pats) and "peak_sustained" not in h and "pct_of_peak" not in h:
            v = row[i]
            try:
                if float(v.replace(",", "")) == 0:
                    continue
            except ValueError:
                pass
            print("   ", h, v, units[i])
