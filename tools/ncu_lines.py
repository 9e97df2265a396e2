"""Aggregate ncu per-SASS metrics to CUDA source lines.
usage: ncu_lines.py <rep> [topN]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
def run(ps):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", ps],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
both = run("cuda,sass")
addr2line, line_src = {}, {}
cur = None; fname = None
for r in both:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) < 4 or r[0] in ("File Path", "Function Name", "Line No"): continue
    if r[0]:
        cur = (fname, int(r[0])); line_src[cur] = r[1][:90]
    elif r[2].startswith("0x") and cur: addr2line[r[2]] = cur
sass = run("sass")
hdr = None; agg = collections.defaultdict(lambda: [0, 0, 0])
for r in sass:
    if len(r) > 5 and r[0] == "Address": hdr = r; ia = r.index("Warp Stall Sampling (All Samples)"); ie = r.index("Instructions Executed"); continue
    if hdr and r and r[0].startswith("0x"):
        ln = addr2line.get(r[0], ("?", 0))
        a = agg[ln]; a[0] += int(r[ia] or 0); a[1] += int(r[ie] or 0); a[2] += 1
tot = sum(v[0] for v in agg.values()); tote = sum(v[1] for v in agg.values())
print(f"total stall samples {tot}, warp instrs {tote}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]*100/tot:5.1f}% samp {v[1]*100/tote:5.1f}% inst  {ln[0]}:{ln[1]:<5} {line_src.get(ln,'')}")
