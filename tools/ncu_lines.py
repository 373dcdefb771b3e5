"""Top source lines by warp-stall samples from an ncu report (--import-source on).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
hdr = None
out = []
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name") and len(r) > 7:
        try:
            st = {hdr[i][6:]: float(r[i]) for i in range(len(hdr))
                  if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i] not in ("0", "")}
            out.append((float(r[4] or 0), f, r[0], r[1][:80], sorted(st.items(), key=lambda x: -x[1])[:3],
                        r[7]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1.0
for o in sorted(out, key=lambda o: -o[0])[:top]:
    stalls = " ".join(f"{k}:{v/o[0]*100:.0f}%" for k, v in o[4]) if o[0] else ""
    print(f"{o[0]/tot*100:5.1f}% {o[1]}:{o[2]:<5} {o[3]:<80} | {stalls} | inst {o[5]}")
