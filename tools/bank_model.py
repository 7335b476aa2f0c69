"""Shared-memory bank model of the hydro stage kernel (csrc/stage_kernel.cuh):
8-byte loads served per half-warp over 16 eight-byte banks; counts the
wavefronts of the face passes' pencil loads (interior positions) for candidate
row / plane pitches, and of the accumulator updates for candidate layouts.
Used for DESIGN §8 (no layout expressible by TMA boxes saves more than a few
per cent of the kernel)."""
import itertools
def face_map(tid, axis):
    warp, lane = tid >> 5, tid & 31
    j = lane % 10; r = lane // 10; p = warp * 10 + j
    if axis == 1: c2, c1 = p & 7, p >> 3
    else: c1, c2 = p & 7, p >> 3
    return (lane < 30 and p < 64), c1, c2, r

def addr(axis, pos, c1, c2, PY, PZ, VS):
    # B0 interior positions only (2..9); faces slabs ignored here
    if axis == 0: x, y, z = pos - 2, c1, c2
    elif axis == 1: x, y, z = c2, pos - 2, c1
    else: x, y, z = c1, c2, pos - 2
    return z * PZ + y * PY + x

def wavefronts(PY, PZ, VS=640, threads=224):
    tot = 0; ideal = 0
    for axis in range(3):
        for w in range(threads // 32):
            for s in range(6):
                for half in range(2):
                    banks = {}
                    n = 0
                    for lane in range(half * 16, half * 16 + 16):
                        act, c1, c2, r = face_map(w * 32 + lane, axis)
                        if not act: continue
                        pos = 3 * r + s
                        if pos < 2 or pos >= 10: continue
                        a = addr(axis, pos, c1, c2, PY, PZ, VS)
                        banks.setdefault(a % 16, set()).add(a)
                        n += 1
                    if n:
                        tot += max(len(v) for v in banks.values())
                        ideal += 1
    return tot, ideal

for PY, PZ in [(10, 80)]:
    print("current", PY, PZ, wavefronts(PY, PZ))
best = []
for PY in range(8, 14):
    for PZ in range(8 * PY, 8 * PY + 24):
        t, i = wavefronts(PY, PZ)
        best.append((t, PY, PZ, i))
best.sort()
print(best[:10])
print("---- even row pitch (TMA inner extent multiple of 16 B), plane pitch mod 16")
res = []
for PY in (8, 10, 12, 14):
    for pzm in range(16):
        PZ = 8 * PY * 5 + ((pzm - 8 * PY * 5) % 16)   # a per-plane layout: plane >= V*8*PY, residue pzm
        t, i = wavefronts(PY, PZ)
        res.append((t, PY, pzm, PZ))
res.sort()
print(res[:8])
print("dense box (PZ = 8*PY):", [(PY, wavefronts(PY, 8 * PY)[0]) for PY in (8, 10, 12, 14)])

# ---- accumulator updates
def cell(axis, c0, c1, c2):
    cc = [0, 0, 0]; cc[axis] = c0; cc[(axis + 1) % 3] = c1; cc[(axis + 2) % 3] = c2
    return (cc[2] * 8 + cc[1]) * 8 + cc[0]
def wf(accf, threads=256):  # accumulator-update wavefronts
    tot = ideal = 0
    for axis in range(3):
        for w in range(threads // 32):
            for k in range(3):
                for half in range(2):
                    banks = {}; n = 0
                    for lane in range(half * 16, half * 16 + 16):
                        act, c1, c2, r = face_map(w * 32 + lane, axis)
                        if not act: continue
                        ncell = 2 if r == 2 else 3
                        if k >= ncell: continue
                        a = accf(cell(axis, 3 * r + k, c1, c2))
                        banks.setdefault(a % 16, set()).add(a); n += 1
                    if n:
                        tot += max(len(v) for v in banks.values()); ideal += 1
    return tot, ideal
print("pitch 8", wf(lambda c: c))
print("pitch 9 (current)", wf(lambda c: (c >> 3) * 9 + (c & 7)))
best = []
for px in range(8, 12):
    for pz in range(0, 16):
        f = lambda c, px=px, pz=pz: (c >> 6) * (8 * px + pz) + ((c >> 3) & 7) * px + (c & 7)
        best.append((wf(f)[0], px, pz))
best.sort(); print(best[:6])
# xor swizzles
for name, f in [("x^y", lambda c: (c & ~7) | ((c & 7) ^ ((c >> 3) & 7))),
                ("x^(y+z)", lambda c: (c & ~7) | ((c & 7) ^ (((c >> 3) + (c >> 6)) & 7))),
                ("x^y, +z*8skew", lambda c: ((c >> 6) * 72) + ((c >> 3) & 7) * 8 + ((c & 7) ^ ((c >> 3) & 7)))]:
    print(name, wf(f))
