"""Top stalled SASS instructions of the first kernel in an `ncu --page source --csv` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
body = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[0].startswith("0x"):
        body.append(r)
S = hdr.index("# Samples")
cols = {k: hdr.index(k) for k in ("Source", "stall_long_sb", "stall_wait", "stall_short_sb",
                                  "stall_math", "stall_not_selected", "Instructions Executed")}
tot = sum(float(r[S]) for r in body)
print("total samples", tot, "instructions", len(body))
idx = sorted(range(len(body)), key=lambda i: -float(body[i][S]))[:top]
for i in sorted(idx):
    r = body[i]
    print(f"#{i:4d} {float(r[S]) / tot * 100:5.1f}% lsb={r[cols['stall_long_sb']]:>6} "
          f"wait={r[cols['stall_wait']]:>6} ssb={r[cols['stall_short_sb']]:>5} "
          f"math={r[cols['stall_math']]:>5} ex={r[cols['Instructions Executed']]:>9} "
          f"{r[cols['Source']].strip()[:90]}")
