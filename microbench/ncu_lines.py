"""Per-source-line warp-stall samples from an ncu report (--print-source cuda,sass):
python microbench/ncu_lines.py REPORT.ncu-rep [top_n]  -> lines sorted by samples, with the
stall-reason columns that dominate each line."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, file, hdr, tot = [], None, None, 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        n = int(r[4])
    except ValueError:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    reasons = {k: int(v) for k, v in zip(hdr, r) if k.startswith("stall_") or "Stall" in k}
    rows.append((n, f"{file}:{r[0]}", r[1][:90], r))
    tot += n
rows.sort(reverse=True)
print(f"total samples {tot}")
for n, loc, src, r in rows[:top]:
    st = sorted(((int(v), k[6:]) for k, v in zip(hdr, r) if k.startswith("stall_") and "Not Issued" not in k
                 and v.isdigit()), reverse=True)[:3]
    why = " ".join(f"{k}:{100.0 * v / max(n, 1):.0f}%" for v, k in st if v)
    print(f"{n:9d} {100.0 * n / tot:5.1f}%  {loc:28s} {src[:70]:70s} [{why}]")
