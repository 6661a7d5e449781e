"""SASS evidence of the Blackwell-native kernels: per kernel of the built
objects, counts of the instructions that prove tcgen05 / TMEM / TMA / bulk
copies / mma.sync / vector memory (cuobjdump -sass on build/*.o).

    python tools/sass_summary.py [tag]   ->  profiles/<tag>_sass.md
"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = [("UTCHMMA", "tcgen05.mma (bf16, TMEM accumulator)"), ("UTCBAR", "tcgen05.commit -> mbarrier"),
       ("LDTM", "tcgen05.ld (TMEM -> registers)"), ("UTMALDG", "TMA tensor load (cp.async.bulk.tensor)"),
       ("UTMAPF", "TMA prefetch"), ("UBLKCP", "bulk copy (cp.async.bulk)"),
       ("SYNCS", "mbarrier ops"), ("HMMA", "mma.sync (bf16, registers)"), ("LDSM", "ldmatrix"),
       ("MUFU.EX2", "exp2 on the MUFU"), ("LDG.E.128", "16-byte global loads"),
       ("STG.E.128", "16-byte global stores"), ("LDG.E.NA.128", "16-byte loads, no L1 allocate")]


def kernels(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            op = m.group(1)
            for key, _ in OPS:
                if op == key or op.startswith(key + "."):
                    counts[cur][key] += 1
    return counts


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    lines = [f"# {tag}: SASS of the built kernels (`cuobjdump -sass build/*.o`, `tools/sass_summary.py`)",
             "", "Counts of the instructions that show which hardware paths each kernel uses:", ""]
    lines += [f"* `{k}`: {d}" for k, d in OPS]
    lines += ["", "| object | kernel | " + " | ".join(k for k, _ in OPS) + " |",
              "|---|---|" + "---:|" * len(OPS)]
    for obj in sorted(glob.glob(os.path.join(ROOT, "build", "akv_*.o"))):
        if "akv_linear" in obj:
            continue
        counts = kernels(obj)
        names = demangle(list(counts))
        for (mang, c), name in zip(counts.items(), names):
            if not any(c.values()):
                continue
            short = re.sub(r"\(.*", "", name).replace("akv::", "")
            lines.append(f"| {os.path.basename(obj)} | `{short}` | " +
                         " | ".join(str(c.get(k, 0)) for k, _ in OPS) + " |")
    path = os.path.join(ROOT, "profiles", f"{tag}_sass.md")
    open(path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
