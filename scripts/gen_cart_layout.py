"""Generates paper_2408_04372_b200/csrc/st_cart_layout.h: the shared-memory
layouts of the Cartesian vmult kernel (st_cart.cuh), chosen by a bank-conflict
model of its four access patterns.

Model: 64-bit shared accesses are served per half-warp; a half-warp costs as
many wavefronts as the largest number of DISTINCT addresses that fall on one
8-byte bank pair (double index mod 16). Lane t of a CTA is (group g, cell c,
a = l % N, b = l / N), l = t % N^2. Offsets are x*1 + y*RY + z*PZ + field*SD
+ cell*CS. Patterns (every one is 2 F N accesses per cell):
  A  store y-lines of layout 1  (x = a, z = b)
  B  load  x-lines of layout 1, store x-lines of layout 2 ((y, z) = (a, b) or
     (b, a) if swapped -- the same for the load and the store)
  C  load  z-lines of layout 2  (x = a, y = b)
Gather (A) and scatter (C) keep lanes along x for coalescing; only the
stage-B line assignment may be swapped. A "split" layout (layout 2 != 1)
needs a barrier between the stage-B loads and stores; it is used only when
it saves wavefronts.

  python scripts/gen_cart_layout.py   (rewrites the header)
"""
import itertools
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cfg(N, F):
    FG = 2 if N * F > 20 else 1
    NC = max(1, 128 // (N * N))
    T = ((NC * N * N * FG + 31) // 32) * 32
    return FG, NC, T


def lanes(N, NC, FG, T):
    out = []
    for w in range(0, T, 32):
        ws = []
        for ln in range(32):
            t = w + ln
            g, r = divmod(t, NC * N * N)
            if g >= FG:
                continue
            c, l = divmod(r, N * N)
            ws.append((ln, c, l % N, l // N))
        out.append(ws)
    return out


def wavefronts(offs):
    tot = 0
    for h in (0, 1):
        cnt = {}
        for ln, d in offs:
            if ln // 16 == h:
                cnt.setdefault(d % 16, set()).add(d)
        if cnt:
            tot += max(len(v) for v in cnt.values())
    return tot


def pattern_cost(L, RY, PZ, CS, kind):
    f = {"y": lambda a, b: a + b * PZ, "x": lambda a, b: a * RY + b * PZ, "xs": lambda a, b: b * RY + a * PZ,
         "z": lambda a, b: a + b * RY}[kind]
    return sum(wavefronts([(ln, c * CS + f(a, b)) for ln, c, a, b in ws]) for ws in L)


def injective_span(N, RY, PZ):
    seen = set()
    for x, y, z in itertools.product(range(N), repeat=3):
        o = x + y * RY + z * PZ
        if o in seen:
            return None
        seen.add(o)
    return max(seen) + 1


def layouts(N):
    """minimal span for every (RY mod 16, PZ mod 16) residue pair"""
    best = {}
    for RY in range(1, 4 * N * N):
        for PZ in range(1, 4 * N * N):
            s = injective_span(N, RY, PZ)
            if s is None or s > 1.35 * N ** 3:
                continue
            k = (RY % 16, PZ % 16)
            if k not in best or s < best[k][2]:
                best[k] = (RY, PZ, s)
    return best


def choose(N, F):
    FG, NC, T = cfg(N, F)
    L = lanes(N, NC, FG, T)
    lay = layouts(N)
    cands = []
    for (ry, pz), (RY, PZ, span) in lay.items():
        for pad in range(16):
            CS = F * span + pad
            c = {k: pattern_cost(L, RY, PZ, CS, k) for k in ("y", "x", "xs", "z")}
            cands.append(((RY, PZ, span, CS), c))
    single = min(((c["y"] + 2 * c[s] + c["z"], lay_[3], lay_, s) for lay_, c in cands for s in ("x", "xs")))
    split = None
    for s in ("x", "xs"):
        l1 = min((c["y"] + c[s], lay_[3], lay_) for lay_, c in cands)
        l2 = min((c[s] + c["z"], lay_[3], lay_) for lay_, c in cands)
        tot = (l1[0] + l2[0], max(l1[1], l2[1]), l1[2], l2[2], s)
        if split is None or tot[:2] < split[:2]:
            split = tot
    ideal = 4 * 2 * (T // 32)
    if split[0] < single[0]:
        return dict(split=1, swap=int(split[4] == "xs"), l1=split[2], l2=split[3], cost=split[0], ideal=ideal,
                    single_cost=single[0])
    return dict(split=0, swap=int(single[3] == "xs"), l1=single[2], l2=single[2], cost=single[0], ideal=ideal,
                single_cost=single[0])


def choose_fdm(N, NT):
    """single in-place layout of the FDM smoother (asm_fdm.cu: fdm_lines_kernel):
    y-lines twice (stages A, E), x-lines four times (B, D), z-lines twice (C)"""
    NC = max(1, 128 // (N * N))
    L = lanes(N, NC, 1, 128)
    best = None
    for (ry, pz), (RY, PZ, span) in layouts(N).items():
        for pad in range(16):
            CS = NT * span + pad
            c = {k: pattern_cost(L, RY, PZ, CS, k) for k in ("y", "x", "xs", "z")}
            for s_ in ("x", "xs"):
                key = (2 * c["y"] + 4 * c[s_] + 2 * c["z"], CS)
                if best is None or key < best[0]:
                    best = (key, (RY, PZ, span, CS), int(s_ == "xs"))
    return best


def main():
    fdm = []
    for N in (2, 3, 4, 5):
        for NT in (1, 2, 3, 4):
            b = choose_fdm(N, NT)
            fdm.append((N, NT, b))
            print("fdm", N, NT, b)
    rows = []
    for N in (2, 3, 4, 5):
        for F in range(1, 9):
            r = choose(N, F)
            rows.append((N, F, r))
            print(N, F, r)
    path = os.path.join(ROOT, "paper_2408_04372_b200", "csrc", "st_cart_layout.h")
    with open(path, "w") as f:
        f.write("// Generated by scripts/gen_cart_layout.py -- shared-memory layouts of the\n"
                "// Cartesian vmult (st_cart.cuh) from a bank-conflict model; do not edit.\n"
                "// Columns: split, swap, RY1, PZ1, SD1, CS1, RY2, PZ2, SD2, CS2,\n"
                "// modelled wavefronts per (field, line point) group / conflict-free ideal.\n"
                "#pragma once\n\nnamespace stmgb {\nnamespace stc {\n\n"
                "template <int N, int F>\nstruct Layout;\n")
        for N, F, r in rows:
            (ry1, pz1, s1, cs1), (ry2, pz2, s2, cs2) = r["l1"], r["l2"]
            f.write(f"template <>\nstruct Layout<{N}, {F}> {{  // {r['cost']} / {r['ideal']} (single layout {r['single_cost']})\n"
                    f"  static constexpr int SPLIT = {r['split']}, SWAP = {r['swap']};\n"
                    f"  static constexpr int RY1 = {ry1}, PZ1 = {pz1}, SD1 = {s1}, CS1 = {cs1};\n"
                    f"  static constexpr int RY2 = {ry2}, PZ2 = {pz2}, SD2 = {s2}, CS2 = {cs2};\n}};\n")
        f.write("\n// FDM smoother (asm_fdm.cu), one in-place layout: SWAP, RY, PZ, SD, CS\n"
                "template <int N, int NT>\nstruct FdmLayout;\n")
        for N, NT, b in fdm:
            (RY, PZ, span, CS), sw = b[1], b[2]
            f.write(f"template <>\nstruct FdmLayout<{N}, {NT}> {{  // {b[0][0]} modelled wavefronts\n"
                    f"  static constexpr int SWAP = {sw}, RY = {RY}, PZ = {PZ}, SD = {span}, CS = {CS};\n}};\n")
        f.write("\n}  // namespace stc\n}  // namespace stmgb\n")


if __name__ == "__main__":
    main()
