"""Count instructions between consecutive barriers of a SASS dump (per-step cost of the sweep
loops).  usage: python tools/sass_loops.py dump.txt"""
import re, sys
lines = [l for l in open(sys.argv[1]) if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
ins = [re.sub(r"\s*/\*[^*]*\*/\s*", " ", l).strip() for l in lines]
bars = [i for i, t in enumerate(ins) if "BAR.SYNC" in t or "BAR.RED" in t]
for a, b in zip(bars, bars[1:]):
    seg = ins[a + 1:b + 1]
    nsq = sum("MUFU.SQRT" in t for t in seg)
    if nsq == 0 and "MUFU.RSQ" not in " ".join(seg):
        continue
    s2r = sum("S2R" in t for t in seg)
    lds = sum(t.split()[0].startswith("LDS") or (len(t.split()) > 1 and t.split()[1].startswith("LDS")) for t in seg)
    ldg = sum("LDG" in t for t in seg)
    print(f"seg {a}-{b}: {len(seg)} instr, sqrt {nsq}, S2R {s2r}, LDS {lds}, LDG {ldg}, end {seg[-1][:40]}")
