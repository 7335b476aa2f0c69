"""Per-kernel SASS mnemonic counts of the product library (cuobjdump -sass):
evidence of what the hot kernels compile to (TMA UTMALDG / UBLKCP, mbarrier
SYNCS, cp.async LDGSTS, DFMA/DMUL/DADD, MUFU) for profiles/."""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2412_15518_b200/libtmgpu.so"
keep = re.compile(r"stage_kernel|amr_m2l|amr_wx|amr_l2p|amr_m2m|amr_mass|pull_kernel|pack_kernel|"
                  r"max_wavespeed|scatter_wavespeed|reflux|grav_correct|stage_epilogue")
watch = ("UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "DFMA", "DMUL", "DADD", "DSETP", "MUFU", "LDS", "STS",
         "LDG", "STG", "SHFL", "BAR", "CALL", "HMMA", "DMMA", "UTCMMA", "UTCBAR")
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1) if keep.search(m.group(1)) else None
        if cur:
            counts[cur] = collections.Counter()
        continue
    if cur:
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            counts[cur][m.group(1)] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
for name, dn in zip(counts, demangle):
    c = counts[name]
    total = sum(c.values())
    shown = "  ".join(f"{k} {sum(v for kk, v in c.items() if kk == k)}" for k in watch if c.get(k))
    print(f"{dn[:110]}\n    {total} instructions: {shown}")
