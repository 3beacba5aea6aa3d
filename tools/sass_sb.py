"""Decode scoreboard control fields from `cuobjdump -sass` output (sm_70+ encoding):
prints, for instructions matching a regex, stall / write-sb / read-sb / wait-mask."""
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else re.compile(".")
lo, hi = (int(x, 0) for x in sys.argv[3].split(":")) if len(sys.argv) > 3 else (0, 1 << 30)
i = 0
while i < len(lines) - 1:
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", lines[i])
    if m:
        m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        if m2:
            addr, text, hiw = int(m.group(1), 16), m.group(2).strip(), int(m2.group(1), 16)
            c = hiw >> 41
            stall, yld, wr, rd, wait = c & 15, (c >> 4) & 1, (c >> 5) & 7, (c >> 8) & 7, (c >> 11) & 63
            if pat.search(text) and lo <= addr <= hi:
                w = ",".join(str(b) for b in range(6) if wait >> b & 1)
                print(f"{addr:05x} st={stall:2d} wr={'-' if wr == 7 else wr} rd={'-' if rd == 7 else rd} "
                      f"wait={{{w}}} {text[:70]}")
            i += 2
            continue
    i += 1
