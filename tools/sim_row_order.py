"""Host simulation of the force sweep's gather locality under list layouts.

For a cfg2-like system (rho = 0.8, r_v = 2.8, cells of side >= r_v, particles
in cell order) it builds the per-particle Verlet rows of a sample of 32-row
warps and counts, per SELL-32 iteration, the distinct 128-byte lines the
warp's 32 float4 gathers touch (the L1 data-pipe cost of the sweep, DESIGN
§11) and the iterations (one coalesced index load each).  Layouts:

  plain     rows in candidate (cell) order, left-aligned (the shipped layout)
  run       each row split by stencil run (9 x-runs of 3 cells), every run
            padded to the warp's longest row in that run
  cell      the same per stencil cell (27)
  greedy    left-aligned (iterations = longest row) but each lane's entries
            permuted: per iteration the lines needed by most still-active lanes
            are served first (a greedy set cover per slot)

Usage: python tools/sim_row_order.py [n_warps] [mode: poisson|lattice]
"""
import sys

import numpy as np

RHO, RV = 0.8, 2.8


def system(mode, key=1):
    g = np.random.default_rng(key)
    a = RHO ** (-1 / 3)
    nx, ny, nz = 128, 128, 64
    L = np.array([nx * a, ny * a, nz * a])
    if mode == "lattice":
        ijk = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
        x = (ijk.reshape(-1, 3) + 0.5 + g.normal(0, 0.15, (nx * ny * nz, 3))) * a
        x %= L
    else:
        x = g.random((nx * ny * nz, 3)) * L
    return x, L


def main():
    nw = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
    mode = sys.argv[2] if len(sys.argv) > 2 else "poisson"
    x, L = system(mode)
    nc = np.floor(L / RV).astype(int)
    cs = L / nc
    c3 = np.minimum((x / cs).astype(int), nc - 1)
    cid = c3[:, 0] + nc[0] * (c3[:, 1] + nc[1] * c3[:, 2])
    g = np.random.default_rng(7)
    order = np.lexsort((g.random(len(x)), cid))
    x, c3, cid = x[order], c3[order], cid[order]
    start = np.searchsorted(cid, np.arange(nc.prod() + 1))
    n = len(x)
    rng = np.random.default_rng(3)
    warps = rng.choice(n // 32, nw, replace=False)
    tot = {k: [0, 0] for k in ("plain", "run", "cell", "greedy", "rank", "pop", "rankpop", "prop", "prop_u", "lead_pop", "lead_low", "first_pop", "greedy_static", "core12", "core16", "core20", "core24", "core28")}
    nbar = 0
    for w in warps:
        rows = []  # per lane: list of (stencil run, stencil cell, j)
        for i in range(w * 32, w * 32 + 32):
            ent = []
            ci = c3[i]
            r = 0
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        cc = (ci + (dx, dy, dz)) % nc
                        c = cc[0] + nc[0] * (cc[1] + nc[1] * cc[2])
                        js = np.arange(start[c], start[c + 1])
                        d = x[js] - x[i]
                        d -= L * np.round(d / L)
                        ok = (np.einsum("ij,ij->i", d, d) < RV * RV) & (js != i)
                        for j in js[ok]:
                            ent.append(((dz + 1) * 3 + dy + 1, r, j))
                        r += 1
            rows.append(ent)
        nbar += sum(len(e) for e in rows)
        # plain: left-aligned rows
        m = max(len(e) for e in rows)
        for t in range(m):
            lines = {e[t][2] >> 3 for e in rows if t < len(e)}
            tot["plain"][0] += len(lines)
        tot["plain"][1] += m
        # key-sorted layouts: each lane sorts its own entries by a key
        pop = {}
        for es in rows:
            for ln in {e[2] >> 3 for e in es}:
                pop[ln] = pop.get(ln, 0) + 1
        for name in ("rank", "pop", "rankpop"):
            srt = []
            for es in rows:
                js = sorted(e[2] for e in es)
                seen = {}
                keyed = []
                for j in js:
                    r = seen.get(j >> 3, 0)
                    seen[j >> 3] = r + 1
                    ln = j >> 3
                    if name == "rank":
                        k = (r, ln)
                    elif name == "pop":
                        k = (-pop[ln], ln, r)
                    else:
                        k = (r, -pop[ln], ln)
                    keyed.append((k, j))
                srt.append([j for _, j in sorted(keyed)])
            for t in range(m):
                tot[name][0] += len({es[t] >> 3 for es in srt if t < len(es)})
            tot[name][1] += m
        # proportional: entry at union position u goes to slot ~ u * m / U
        for name in ("prop", "prop_u"):
            allj = sorted({e[2] for es in rows for e in es})
            if name == "prop_u":  # union position measured in lines
                lines_u = sorted({j >> 3 for j in allj})
                pos = {j: lines_u.index(j >> 3) + (j & 7) / 8.0 for j in allj}
                U = len(lines_u)
            else:
                pos = {j: q for q, j in enumerate(allj)}
                U = len(allj)
            slots = {}
            for es in rows:
                js = sorted(e[2] for e in es)
                L_ = len(js)
                sl = []
                prev = -1
                for q, j in enumerate(js):
                    tgt = int(pos[j] * m / U)
                    tgt = max(prev + 1, min(tgt, m - (L_ - q)))
                    sl.append(tgt)
                    prev = tgt
                for t, j in zip(sl, js):
                    slots.setdefault(t, set()).add(j >> 3)
            tot[name][0] += sum(len(v) for v in slots.values())
            tot[name][1] += m
        # leader rounds: per slot, a leader lane picks a line; every unserved
        # lane holding an entry on it takes one; repeat until all are served
        for name in ("lead_pop", "lead_low", "first_pop", "greedy_static"):
            rem = [sorted(e[2] for e in es) for es in rows]
            its = 0
            while any(rem):
                todo = {k for k in range(32) if rem[k]}
                nl = 0
                while todo:
                    if name == "greedy_static":
                        cand = {j >> 3 for k in todo for j in rem[k]}
                        best = max(cand, key=lambda q: (pop[q], -q))
                    else:
                        if name == "first_pop":
                            ld = min(todo)
                        else:
                            ld = max(todo, key=lambda k: (len(rem[k]), -k))
                        lines_ld = {j >> 3 for j in rem[ld]}
                        if name == "lead_low":
                            best = min(lines_ld)
                        else:
                            best = max(lines_ld, key=lambda q: (pop[q], -q))
                    nl += 1
                    for k in list(todo):
                        for t, j in enumerate(rem[k]):
                            if j >> 3 == best:
                                del rem[k][t]
                                todo.discard(k)
                                break
                tot[name][0] += nl
                its += 1
            tot[name][1] += its
        # core + backfill: lines needed by >= thr lanes get aligned slot blocks
        # (max multiplicity over lanes); the other entries fill the holes, then
        # append
        for thr in (12, 16, 20, 24, 28):
            core = sorted(q for q in pop if pop[q] >= thr)
            base = {}
            o = 0
            for q in core:
                base[q] = o
                o += max(sum(1 for e in es if e[2] >> 3 == q) for es in rows)
            slots = {}
            its = 0
            for es in rows:
                js = sorted(e[2] for e in es)
                used = set()
                rest = []
                cnt = {}
                for j in js:
                    q = j >> 3
                    if q in base:
                        t = base[q] + cnt.get(q, 0)
                        cnt[q] = cnt.get(q, 0) + 1
                        used.add(t)
                        slots.setdefault(t, set()).add(q)
                    else:
                        rest.append(j)
                t = 0
                for j in rest:
                    while t in used:
                        t += 1
                    used.add(t)
                    slots.setdefault(t, set()).add(j >> 3)
                its = max(its, max(used) + 1 if used else 0)
            tot[f"core{thr}"][0] += sum(len(v) for v in slots.values())
            tot[f"core{thr}"][1] += its
        # greedy: per slot, serve the most popular line among active lanes
        rem = [sorted(e[2] for e in es) for es in rows]
        its = 0
        while any(rem):
            act = [k for k in range(32) if rem[k]]
            todo = set(act)
            nl = 0
            while todo:
                cnt = {}
                for k in todo:
                    for ln in {j >> 3 for j in rem[k]}:
                        cnt[ln] = cnt.get(ln, 0) + 1
                best = max(cnt, key=lambda q: (cnt[q], -q))
                nl += 1
                for k in list(todo):
                    for t, j in enumerate(rem[k]):
                        if j >> 3 == best:
                            del rem[k][t]
                            todo.discard(k)
                            break
            tot["greedy"][0] += nl
            its += 1
        tot["greedy"][1] += its
        for key, idx in (("run", 0), ("cell", 1)):
            groups = sorted({e[idx] for es in rows for e in es})
            for gk in groups:
                sub = [[e for e in es if e[idx] == gk] for es in rows]
                mm = max(len(s) for s in sub)
                for t in range(mm):
                    lines = {s[t][2] >> 3 for s in sub if t < len(s)}
                    tot[key][0] += len(lines)
                tot[key][1] += mm
    print(f"{mode}: {nw} warps, mean row {nbar / (32 * nw):.2f}")
    for k, (lines, its) in tot.items():
        print(f"  {k:6s} iterations/warp {its / nw:7.2f}  lines/iteration {lines / its:6.2f}"
              f"  lines+index wavefronts per warp {(lines + its) / nw:8.1f}")


if __name__ == "__main__":
    main()
