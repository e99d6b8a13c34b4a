"""Count tcgen05 / TMA SASS instructions per kernel of the built library
(cuobjdump -sass) -> profiles/r1_sass_evidence.txt."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2201_05596_b200/libmoe_b200.so"
out_path = sys.argv[2] if len(sys.argv) > 2 else "profiles/r1_sass_evidence.txt"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMACCTL", "LDTM", "UTCATOMSWS",
        "SYNCS.EXCH", "SYNCS.ARRIVE", "UCGABAR", "ELECT", "MATCH", "REDG"]
funcs = re.split(r"\n\s*Function : ", txt)
rows, tot = [], collections.Counter()
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    c = collections.Counter({k: len(re.findall(r"\b" + re.escape(k), f)) for k in keys})
    if any(c[k] for k in ("UTCHMMA", "UTMALDG", "LDTM", "UTMASTG")):
        rows.append((name[:90], {k: v for k, v in c.items() if v}))
    tot.update(c)
out = ["tcgen05 / TMA evidence in libmoe_b200.so (cuobjdump -sass, sm_100a); instruction counts "
       "per kernel", ""]
for n, c in rows:
    out.append(f"{n}\n    {c}")
out += ["", f"kernels with tcgen05/TMA: {len(rows)} of {len(funcs) - 1}; totals: "
        f"{ {k: v for k, v in tot.items() if v} }"]
open(out_path, "w").write("\n".join(out) + "\n")
print(out[-1])
