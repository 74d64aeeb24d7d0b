"""Per-kernel SASS instruction counts of the built tensor-core objects (cuobjdump -sass), as evidence
that the conv passes are tcgen05 / TMA / TMEM kernels: UTCHMMA (tcgen05.mma, .2CTA = cta_group::2),
UTMALDG (TMA tensor loads), LDTM (tcgen05.ld TMEM -> registers), UTCBAR (tcgen05.commit), plus the
peer-memory / synchronisation instructions of the fused collectives.  Writes a text table.

usage: python scripts/sass_summary.py [out.txt]   (after paper_1712_02546_b200/build.py)"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_1712_02546_b200", "build")
# instruction families reported with their full mnemonics (e.g. UTMALDG.4D.2CTA)
FAMILIES = ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMAPF", "LDTM", "UTCBAR", "UTCATOM", "RED", "ATOMG", "MEMBAR",
            "FENCE", "NANOSLEEP", "HMMA")


def demangle(name):
    r = subprocess.run(["c++filt", name], capture_output=True, text=True)
    return r.stdout.strip() or name


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    lines = []
    for obj in ("kernels_tc.cu.o", "kernels_conv1.cu.o", "kernels_simt.cu.o", "comm.cu.o"):
        path = os.path.join(OBJ, obj)
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        cur, counts = None, collections.OrderedDict()
        for ln in sass.splitlines():
            m = re.search(r"Function : (\S+)", ln)
            if m:
                cur = demangle(m.group(1))
                counts[cur] = collections.Counter()
                continue
            if cur is None:
                continue
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]+)", ln)
            if not m:
                continue
            op = m.group(2)
            counts[cur]["instructions"] += 1
            if op.split(".")[0] in FAMILIES:
                counts[cur][op] += 1
        for fn, c in counts.items():
            fam = {k: v for k, v in c.items() if k != "instructions"}
            if obj not in ("kernels_tc.cu.o", "kernels_conv1.cu.o") and not fam:
                continue
            short = re.sub(r"cp::\(anonymous namespace\)::|\(anonymous namespace\)::|cp::", "", fn).split("(")[0]
            items = ", ".join(f"{k} {v}" for k, v in sorted(fam.items()))
            lines.append(f"{obj:18s} {short:40s} {c['instructions']:6d} instr | {items}")
    text = ("# cuobjdump -sass instruction counts per kernel (sm_100a build of this commit)\n"
            "# conv_tc_kernel<PASS, CG, DT>: PASS 0 fwd / 1 dgrad / 2 wgrad; CG 2 = CTA pair (cta_group::2); "
            "DT 1 = bf16 operands\n" + "\n".join(lines) + "\n")
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
