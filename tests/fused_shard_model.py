"""Model (plain Python, CPU) of the sharded fused protocol of
csrc/fused_shard.cuh, for the gloo multi-process tests: the same slot
contents (exchange 1: Bic header + final stack with chunk-local contexts;
exchange 2: chunk union, su of each final-stack open, the closes of imported
entries with this chunk's part of their union) and the same compose / fix-up
arithmetic (sh_table, imported_ctx, sh_fixup), with the chunk-local passes done
by a sequential stack walk (Fig. 1; the oracle's box rules R2-R10)
instead of the tile kernels.  Test infrastructure only."""
import numpy as np

F = np.float32
INF = np.array([-np.inf, -np.inf, np.inf, np.inf], F)
EMPTY = np.array([np.inf, np.inf, -np.inf, -np.inf], F)
OPEN_CLIP, OPEN_BLEND, CLOSE = 1, 2, 3


def isect(a, b):
    return np.concatenate([np.maximum(a[:2], b[:2]), np.minimum(a[2:], b[2:])]).astype(F)


def unite(a, b):
    return np.concatenate([np.minimum(a[:2], b[:2]), np.maximum(a[2:], b[2:])]).astype(F)


def phase1(tags, boxes, goff):
    """Slot 1 of a chunk: (a, b) and its final stack bottom to top: global
    index | blend << 31, the context its children see inside the chunk (INF
    below the chunk start)."""
    stack, a = [], 0
    for i, t in enumerate(tags):
        ctx = stack[-1][1] if stack else INF
        if t == OPEN_CLIP:
            stack.append(((goff + i), isect(boxes[i], ctx)))
        elif t == OPEN_BLEND:
            stack.append(((goff + i) | (1 << 31), ctx))
        elif t == CLOSE:
            if stack:
                stack.pop()
            else:
                a += 1
    idx = [np.int32(np.uint32(s[0]).view(np.int32)) for s in stack]
    return {"a": a, "b": len(stack), "idx": idx, "lcc": [s[1] for s in stack]}


def table(slots1):
    """sh_table: start height H, low-water L per chunk; tcc = the context
    below each chunk's final stack (F1 over chunks)."""
    tab, H = [], 0
    for s in slots1:
        L = max(H - s["a"], 0)
        tab.append((H, L, s["a"], s["b"]))
        H = L + s["b"]
    tcc = []
    for k in range(len(slots1)):
        X = tab[k][1] - 1
        c = INF
        if X >= 0:
            j = owner_chunk(tab, k, X)
            c = isect(slots1[j]["lcc"][X - tab[j][1]], tcc[j])
        tcc.append(c)
    return tab, tcc


def owner_chunk(tab, k, X):
    for j in range(k - 1, -1, -1):
        if tab[j][1] <= X:
            return j
    return -1


def phase2(tags, boxes, goff, g, slots1):
    """The chunk's walk from its imported stack (the top a + 1 entries of the
    global stack at its start; heights below 0 are root slots).  Returns the
    outputs so far and slot 2."""
    tab, tcc = table(slots1)
    H, _, a, _ = tab[g]
    n = len(tags)
    stack = []  # [kind, open index or -1, ctx, union, imported height or None]
    for X in range(H - a - 1, H):
        if X < 0:
            stack.append(["root", -1, INF, EMPTY.copy(), X])
        else:
            j = owner_chunk(tab, g, X)
            s = slots1[j]
            si = int(s["idx"][X - tab[j][1]])
            stack.append(["imp", si, isect(s["lcc"][X - tab[j][1]], tcc[j]), EMPTY.copy(), X])
    match = np.full(n, -1, np.int32)
    parent = np.full(n, -1, np.int32)
    out = np.zeros((n, 4), F)
    records = {}  # imported height X -> (global close index, this chunk's part of the union)
    cu = EMPTY.copy()
    for i, t in enumerate(tags):
        top = stack[-1] if stack else ["root", -1, INF, EMPTY.copy(), None]
        ptop = -1 if top[0] == "root" else top[1] & 0x7fffffff
        if t == OPEN_CLIP or t == OPEN_BLEND:
            parent[i] = ptop
            if t == OPEN_CLIP:
                c = isect(boxes[i], top[2])
                out[i] = c
                stack.append(["loc", (goff + i), c, EMPTY.copy(), None])
            else:
                out[i] = EMPTY
                stack.append(["loc", (goff + i) | (1 << 31), top[2], EMPTY.copy(), None])
        elif t == CLOSE:
            if not stack or stack[-1][0] == "root":
                if stack:
                    stack.pop()
                out[i] = EMPTY  # R3
                continue
            e = stack.pop()
            o = e[1] & 0x7fffffff
            parent[i] = match[i] = o
            out[i] = e[3]
            if e[0] == "loc":
                match[o - goff] = goff + i
                if e[1] >> 31:
                    out[o - goff] = e[3]
            else:
                records[e[4]] = (goff + i, e[3].copy())
            if stack:
                stack[-1][3] = unite(stack[-1][3], e[3])
        else:
            parent[i] = ptop
            c = isect(boxes[i], top[2])
            out[i] = c
            cu = unite(cu, c)
            if stack:  # the top's union; enclosing ones receive it at its close
                stack[-1][3] = unite(stack[-1][3], c)
    # su: union after each final-stack open to the chunk end = its walk union
    # plus the unions of the entries above it (added at their closes, or still open)
    fin = [s for s in stack if s[0] == "loc"]
    su, acc = [None] * len(fin), EMPTY.copy()
    for k in range(len(fin) - 1, -1, -1):
        acc = unite(acc, fin[k][3])
        su[k] = acc
    return match, parent, out, {"cu": cu, "su": su, "rec": records}, tab


def phase3(g, goff, slots1, slots2, tab, match, out):
    """sh_fixup: nodes spanning chunks."""
    G = len(slots1)

    def cus(a, b):
        u = EMPTY.copy()
        for k in range(a, b + 1):
            u = unite(u, slots2[k]["cu"])
        return u
    # A: this chunk's closes of imported entries
    for X, (c, U) in slots2[g]["rec"].items():
        j = owner_chunk(tab, g, X)
        out[c - goff] = unite(unite(U, slots2[j]["su"][X - tab[j][1]]), cus(j + 1, g - 1))
    # B: later chunks' closes of this chunk's final-stack opens
    for k in range(g + 1, G):
        for X, (c, U) in slots2[k]["rec"].items():
            if owner_chunk(tab, k, X) != g:
                continue
            pos = X - tab[g][1]
            si = int(slots1[g]["idx"][pos])
            o = (si & 0x7fffffff) - goff
            match[o] = c
            if si < 0:
                out[o] = unite(unite(U, slots2[g]["su"][pos]), cus(g + 1, k - 1))
    # C: final-stack opens never closed: blend opens take the union to the end (R4)
    later = min([tab[k][1] for k in range(g + 1, G)], default=1 << 62)
    for pos in range(tab[g][3]):
        X = tab[g][1] + pos
        si = int(slots1[g]["idx"][pos])
        if X < later and si < 0:
            out[(si & 0x7fffffff) - goff] = unite(slots2[g]["su"][pos], cus(g + 1, G - 1))


def protocol(tags, boxes, goff, g, allgather):
    """One rank: two all-gathers (allgather(obj) -> list over ranks)."""
    slots1 = allgather(phase1(tags, boxes, goff))
    match, parent, out, slot2, tab = phase2(tags, boxes, goff, g, slots1)
    slots2 = allgather(slot2)
    phase3(g, goff, slots1, slots2, tab, match, out)
    return match, parent, out
