"""Print the SASS hot loop (around the DMMAs) of one K1 variant: python tools/sass_loop.py BN CONJ"""
import re, subprocess, sys
bn, conj = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", "paper_1206_3768_b200/libchfsi.so"], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if "cheb_step_kernel" in name and f"ILi{bn}E" in name and f"Lb{conj}E" in name:
        ins = [re.sub(r"/\*[0-9a-f]{4,}\*/", "", l).strip().rstrip(";").strip()
               for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
        idx = [i for i, l in enumerate(ins) if "DMMA" in l]
        print(name[:120], "instructions", len(ins), "DMMA", len(idx))
        from collections import Counter
        c = Counter(l.split()[0] if not l.startswith("@") else l.split()[1] for l in ins[idx[0]:idx[-1]])
        print("between first/last DMMA:", c.most_common(12))
        lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
        for l in ins[idx[0] - 5 + lo: idx[0] + 60 + lo]:
            print("   ", l)
        break
