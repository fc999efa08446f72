"""Summarise an ncu report by CUDA source line: top lines by warp-stall samples
with their dominant stall reasons (needs -lineinfo builds and --import-source on)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
cur_file = ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    try:
        samples = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    except ValueError:
        continue
    stalls = {k: float(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-")}
    lines.append((samples, cur_file, r[0], r[1][:90], stalls))
tot = sum(l[0] for l in lines) or 1
lines.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for s, f, ln, src, st in lines[:top]:
    best = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    bs = " ".join(f"{k[6:]}={100*v/max(s,1):.0f}%" for k, v in best)
    print(f"{100*s/tot:5.1f}% {f}:{ln:>5} {src:<90} [{bs}]")
