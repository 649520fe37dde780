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
