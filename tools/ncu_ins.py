import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 80
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
lines = []; file_ = None
for r in rows:
    if r and r[0] == "File Path": file_ = r[1].split("/")[-1]
    if len(r) != len(hdr) or not r[0] or r[0] == "Line No": continue
    try: lines.append((int(r[iI]), int(r[iS]), f"{file_}:{r[0]}", r[1].strip()[:100]))
    except ValueError: pass
ts = sum(x[1] for x in lines) or 1; ti = sum(x[0] for x in lines) or 1
print(f"total samples {ts}, warp instructions {ti}")
for i, s, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*i/ti:5.1f}% ins {100*s/ts:5.1f}% smp  {loc:24s} {src}")
