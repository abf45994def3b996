"""Per-source-line instruction + stall-sample shares from an ncu report (needs -lineinfo)."""
import collections, csv, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = cur_line = None
src, stats = {}, collections.defaultdict(lambda: [0, 0])
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0] != "":
        cur_line = int(r[0]); src[(cur_file, cur_line)] = r[1]
        continue
    try:
        stats[(cur_file, cur_line)][0] += int(r[7]); stats[(cur_file, cur_line)][1] += int(r[4])
    except ValueError:
        pass
ti = sum(v[0] for v in stats.values()); ts = sum(v[1] for v in stats.values())
print(f"total instructions {ti}  stall samples {ts}")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1]/ts:6.1%} samp {v[0]/ti:6.1%} inst  {k[0]}:{k[1]:<5d} {src.get(k, '')[:80]}")
