"""Aggregates an ncu report's SASS-level counters by CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep [top_n]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None; hdr = None; items = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            items.append((cur, int(r[0]), r[1].strip()[:88], int(d["Instructions Executed"]), int(d["# Samples"]),
                          int(d.get("L1 Wavefronts Shared", "0") or 0), int(d.get("L2 Theoretical Sectors Global", "0") or 0)))
        except (ValueError, KeyError):
            pass
ti = sum(i[3] for i in items) or 1; ts = sum(i[4] for i in items) or 1
print(f"total warp instr {ti}  samples {ts}")
for i in sorted(items, key=lambda x: -x[4])[:top]:
    print(f"{i[0]:14s}:{i[1]:4d} {i[3]/ti*100:5.1f}%i {i[4]/ts*100:5.1f}%s shw {i[5]:>10d} l2s {i[6]:>10d}  {i[2]}")
