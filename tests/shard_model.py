"""CPU model of the multi-GPU shard protocol (tests only).

Mirrors paper_2205_11659_b200/csrc/shard.cu step by step with plain Python
stack walks, so the host-side logic of the protocol — chunk summaries (Bic
value + unmatched opens, §3-§4), the owner rule over chunks, the
composed incoming stack, (open, close) pairs routed back to the owning chunk —
can be exercised with real torch.distributed collectives (gloo) on CPU and
checked against the oracle.  It does not import oracle/ or the CUDA path.
"""
from __future__ import annotations

OPEN = (1, 2)
CLOSE = 3


def chunk_summary(tags, off):
    """Bic (a, b) of the chunk and its unmatched opens (global indices)."""
    stack, a = [], 0
    for i, t in enumerate(tags):
        if t in OPEN:
            stack.append(off + i)
        elif t == CLOSE:
            if stack:
                stack.pop()
            else:
                a += 1
    return a, len(stack), stack


def bic_combine(x, y):
    m = min(x[1], y[0])
    return (x[0] + y[0] - m, x[1] + y[1] - m)


def compose(hdrs, opens, g):
    """Top a_g + 1 entries of the stack at chunk g's start: dict height -> index.

    The entry at height X belongs to the last chunk h < g whose low-water mark
    L_h = max(H_h - a_h, 0) <= X, at position X - L_h of its open list."""
    pre = (0, 0)
    L, Hs = [], []
    for h, (a, b) in enumerate(hdrs):
        Hs.append(pre[1])
        L.append(max(pre[1] - a, 0))
        pre = bic_combine(pre, (a, b))
    H = Hs[g]
    lo = max(H - 1 - hdrs[g][0], 0)
    stack = {}
    for X in range(lo, H):
        h = g - 1
        while h > 0 and L[h] > X:
            h -= 1
        stack[X] = opens[h][X - L[h]]
    return H, lo, stack


def finish_chunk(tags, off, H, stack):
    """Stack walk of the chunk starting from the composed stack (heights
    [lo, H) known).  Returns parent, match (chunk-local arrays, global values)
    and the (open, close) pairs for opens of earlier chunks."""
    n = len(tags)
    parent = [-1] * n
    match = [-1] * n
    local = []          # opens pushed inside this chunk (global indices)
    depth_in = 0        # entries of the incoming stack popped so far
    pairs = []
    for i, t in enumerate(tags):
        g = off + i
        if local:
            top = local[-1]
        else:
            X = H - 1 - depth_in
            top = stack[X] if X >= 0 else -1
        parent[i] = top
        if t in OPEN:
            local.append(g)
        elif t == CLOSE:
            if local:
                o = local.pop()
                match[i] = o
                match[o - off] = g
            elif top >= 0:
                match[i] = top
                pairs.append((top, g))
                depth_in += 1
    return parent, match, pairs


def apply_pairs(match, off, all_pairs):
    for o, c in all_pairs:
        if off <= o < off + len(match):
            match[o - off] = c


def protocol(tags_chunk, off, rank, allgather):
    a, b, opens = chunk_summary(tags_chunk, off)
    hdrs = allgather((a, b))
    all_opens = allgather(opens)
    H, lo, stack = compose(hdrs, all_opens, rank)
    parent, match, pairs = finish_chunk(tags_chunk, off, H, stack)
    all_pairs = [p for lst in allgather(pairs) for p in lst]
    apply_pairs(match, off, all_pairs)
    return parent, match


# ---------------------------------------------------------------------------
# tree_bbox shard protocol (mirrors the bbm shard path of csrc/shard.cu):
# inputs are the chunk's tags / boxes and paren_match's GLOBAL parent / match
# for the chunk's elements.  Boxes are (x0, y0, x1, y1) tuples of floats;
# intersection = max/max/min/min, union = min/min/max/max (DESIGN R9-R11).
# ---------------------------------------------------------------------------
INF_BOX = (-float("inf"), -float("inf"), float("inf"), float("inf"))
EMPTY_BOX = (float("inf"), float("inf"), -float("inf"), -float("inf"))


def isect(a, b):
    return (max(a[0], b[0]), max(a[1], b[1]), min(a[2], b[2]), min(a[3], b[3]))


def unite(a, b):
    return (min(a[0], b[0]), min(a[1], b[1]), max(a[2], b[2]), max(a[3], b[3]))


def _contexts(tags, boxes, parent, off, ext):
    """Clip context of every element: box ∩ ctx(parent) (clip opens and leaves),
    ctx(parent) for blend opens; a parent in an earlier chunk takes ext[parent]
    (INF when ext is None: the chunk-local frame)."""
    n = len(tags)
    ctx = [None] * n
    for i in range(n):
        t = tags[i]
        if t == CLOSE:
            continue
        p = parent[i]
        if p < 0:
            pc = INF_BOX
        elif p < off:
            pc = ext.get(p, INF_BOX) if ext is not None else INF_BOX
        else:
            pc = ctx[p - off]
        ctx[i] = pc if t == 2 else isect(tuple(boxes[i]), pc)
    return ctx


def bbox_phase1(tags, boxes, parent, match, off):
    """Final stack of the chunk (opens closed after it or never) with chunk-local
    cumulative clips, and the chunk's link."""
    n = len(tags)
    lctx = _contexts(tags, boxes, parent, off, None)
    fs = [(off + i, lctx[i]) for i in range(n) if tags[i] in OPEN and (match[i] < 0 or match[i] >= off + n)]
    link = parent[fs[0][0] - off] if fs else -1
    return {"off": off, "n": n, "link": link, "fs": fs}


def bbox_compose(summaries, g):
    """True contexts of the final-stack opens of chunks before g (chain over chunks)."""
    tcc = []
    for h, sm in enumerate(summaries):
        t = INF_BOX
        if sm["link"] >= 0:
            h2 = max(k for k in range(h) if summaries[k]["off"] <= sm["link"])
            t = isect(dict(summaries[h2]["fs"])[sm["link"]], tcc[h2])
        tcc.append(t)
    ext = {}
    for h in range(g):
        for idx, v in summaries[h]["fs"]:
            ext[idx] = isect(v, tcc[h])
    return ext


def bbox_phase2(tags, boxes, parent, match, off, ext):
    """Local outputs, the chunk's exports (union, union after each final-stack
    open) and the closes of earlier chunks' nodes with their prefix unions."""
    n = len(tags)
    ctx = _contexts(tags, boxes, parent, off, ext)
    out = [None] * n
    leaf = [tags[i] not in OPEN and tags[i] != CLOSE for i in range(n)]
    for i in range(n):
        if leaf[i] or tags[i] == 1:
            out[i] = ctx[i]

    def seg(a, b):  # union of clipped leaves in [a, b) (local)
        u = EMPTY_BOX
        for j in range(a, b):
            if leaf[j]:
                u = unite(u, out[j])
        return u

    reports = []
    for i in range(n):
        if tags[i] != CLOSE:
            continue
        o = match[i]
        if o < 0:
            out[i] = EMPTY_BOX
        elif o >= off:
            u = seg(o - off + 1, i)
            out[i] = u
            if tags[o - off] == 2:
                out[o - off] = u
        else:
            reports.append((off + i, o, seg(0, i)))
    suc = [(idx, seg(idx - off + 1, n)) for idx, _ in bbox_phase1(tags, boxes, parent, match, off)["fs"]]
    never = [i for i in range(n) if tags[i] == 2 and match[i] < 0]
    for i in never:
        out[i] = seg(i + 1, n)
    return out, {"tu": seg(0, n), "suc": suc, "reports": reports}, never


def bbox_fixup(out, tags, off, g, summaries, exports, never):
    G = len(exports)

    def chunks(a, b):
        u = EMPTY_BOX
        for h in range(a, b + 1):
            u = unite(u, exports[h]["tu"])
        return u

    for c, o, pre in exports[g]["reports"]:
        h = max(k for k in range(G) if summaries[k]["off"] <= o)
        u = unite(unite(pre, chunks(h + 1, g - 1)), dict(exports[h]["suc"]).get(o, EMPTY_BOX))
        out[c - off] = u
    mine = dict(exports[g]["suc"])
    for k in range(g + 1, G):
        for c, o, pre in exports[k]["reports"]:
            if off <= o < off + len(tags) and tags[o - off] == 2:
                out[o - off] = unite(unite(pre, chunks(g + 1, k - 1)), mine.get(o, EMPTY_BOX))
    later = chunks(g + 1, G - 1)
    for i in never:
        out[i] = unite(out[i], later)
    return out


def bbox_protocol(tags, boxes, parent, match, off, rank, allgather):
    summaries = allgather(bbox_phase1(tags, boxes, parent, match, off))
    ext = bbox_compose(summaries, rank)
    out, exp, never = bbox_phase2(tags, boxes, parent, match, off, ext)
    exports = allgather(exp)
    return bbox_fixup(out, tags, off, rank, summaries, exports, never)
