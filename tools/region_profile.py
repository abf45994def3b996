"""Instruction / stall-sample shares of an ncu --set full replay_kernel report by
code region of csrc/replay.cu (function line ranges found by name)."""
import collections, csv, re, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = open("paper_2602_03921_b200/csrc/replay.cu").read().splitlines()
starts = [(i + 1, m.group(1)) for i, l in enumerate(src)
          for m in [re.match(r"(?:DFI|template|__global__)[^(]*?\b(\w+)\(", l)] if m]
def region(line):
    name = "top"
    for ln, n in starts:
        if ln <= line: name = n
    return name
cur_file = cur_line = None
stats = collections.defaultdict(lambda: [0, 0])
lines = collections.defaultdict(lambda: [0, 0])
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if len(r) < 8 or r[0] == "Line No": continue
    if r[0] != "":
        cur_line = int(r[0]); continue
    try:
        i, smp = int(r[7]), int(r[4])
    except ValueError:
        continue
    key = region(cur_line) if cur_file == "replay.cu" else cur_file
    stats[key][0] += i; stats[key][1] += smp
    lines[(cur_file, cur_line)][0] += i; lines[(cur_file, cur_line)][1] += smp
ti = sum(v[0] for v in stats.values()); ts = sum(v[1] for v in stats.values())
print(f"total instructions {ti}  samples {ts}")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {k:28s} inst {v[0]/ti:6.1%}  samples {v[1]/ts:6.1%}")
print("top lines by instructions")
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:40]:
    txt = src[k[1] - 1].strip()[:70] if k[0] == "replay.cu" else ""
    print(f"  {v[0]/ti:6.1%} inst {v[1]/ts:6.1%} samp  {k[0]}:{k[1]}  {txt}")
