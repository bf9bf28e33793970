import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
res = collections.Counter(); st = collections.Counter(); src = {}
f = None; hdr = None
g = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
for row in csv.reader(out.splitlines()):
    if not row: continue
    if row[0] == "File Path": f = row[1].split('/')[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or not row[0].isdigit(): continue
    key = (f, int(row[0])); src[key] = row[1][:80]
    res[key] += g(row[hdr.index("Instructions Executed")]); st[key] += g(row[hdr.index("Warp Stall Sampling (All Samples)")])
tot = sum(st.values())
print("stall samples", tot)
for key, v in sorted(st.items(), key=lambda x: -x[1])[:int(sys.argv[2])]:
    print(f"{key[0]}:{key[1]:4d} stall {100*v/tot:5.1f}% inst {res[key]:>10d}  {src[key]}")
