/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct sequential CPU implementation of what the
 * hot path computes, written from the paper (arXiv 2205.11659, R. Levien,
 * "Fast GPU bounding boxes on tree-structured scenes").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, headers, tables or helpers with
 * the CUDA path (paper_2205_11659_b200/csrc), and the CUDA path never loads it.
 *
 * Citations: P:n = PAPER.md line n (section in brackets).
 * Readings of silent / ambiguous points are numbered as in DESIGN.md §3.
 *
 * Element tags (one byte per element of the flattened tree):
 *   1 = open of a clip node, 2 = open of a blend node, 3 = close,
 *   anything else (0 canonical) = leaf                     [DESIGN R2]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { TAG_OPEN_CLIP = 1, TAG_OPEN_BLEND = 2, TAG_CLOSE = 3 };

/* ------------------------------------------------------------------------ */
/* oracle_paren_match                                                        */
/*                                                                           */
/* Fig. 1 (§2) run literally:                                       */
/*     stack = [-1]                                                          */
/*     for i in range(len(s)):                                               */
/*         out[i] = stack[len(stack) - 1]                                    */
/*         if inp[i] == '(':  stack.push(i)                                  */
/*         elif inp[i] == ')': stack.pop()                                   */
/* parent[i] := out[i]  (the "stronger" problem).                      */
/* match[i]  := classical partner ("traditional version"), -1 if none. */
/* A close that finds only the -1 sentinel (Fig. 1 would pop the sentinel;   */
/* undefined in the paper) leaves the stack unchanged and gets match = -1:   */
/* the stack-monoid semantics of §4, DESIGN R3.                  */
/* Leaves read the top and neither push nor pop (DESIGN R2).                */
/* Returns 0, or -1 on allocation failure.                                   */
/* ------------------------------------------------------------------------ */
int oracle_paren_match(const uint8_t *tags, int64_t n, int32_t *match, int32_t *parent)
{
    int64_t *stack = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    if (!stack) return -1;
    int64_t sp = 0;
    stack[sp++] = -1;
    for (int64_t i = 0; i < n; i++) {
        parent[i] = (int32_t)stack[sp - 1];
        match[i] = -1;
        uint8_t t = tags[i];
        if (t == TAG_OPEN_CLIP || t == TAG_OPEN_BLEND) {
            stack[sp++] = i;
        } else if (t == TAG_CLOSE) {
            if (stack[sp - 1] != -1) {
                int64_t o = stack[--sp];
                match[i] = (int32_t)o;                  /* P:74 partner */
                match[o] = (int32_t)i;
            }                                            /* else: R3 */
        }
    }
    free(stack);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Bounding-box algebra (§6).                                   */
/* Boxes are (x0, y0, x1, y1) fp32.  Intersection = (max x0, max y0, min x1, */
/* min y1); union = (min x0, min y0, max x1, max y1) — raw, never            */
/* canonicalised (DESIGN R9).  min/max (DESIGN R12): ordinary order with     */
/* -0 below +0; a NaN operand is ignored (the other operand is returned),    */
/* and two NaNs give the canonical NaN 0x7fffffff — IEEE 754-2008 minNum /   */
/* maxNum with signed zeros ordered.  NaN is outside the input domain; the   */
/* rule only makes every result a unique bit pattern.                        */
/* ------------------------------------------------------------------------ */
typedef struct { float x0, y0, x1, y1; } box_t;

static uint32_t f32_bits(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static float bits_f32(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }
static int is_nan(float x) { return (f32_bits(x) & 0x7fffffffu) > 0x7f800000u; }

/* x ordered at or below y, for non-NaN x, y: numeric order, and -0 < +0. */
static int ordered_le(float x, float y)
{
    if (x < y) return 1;
    if (x > y) return 0;
    /* equal: only the zeros can differ in bits */
    return (f32_bits(x) >> 31) >= (f32_bits(y) >> 31);   /* -0 <= +0, x == x */
}
static float tmin(float x, float y)
{
    if (is_nan(x) && is_nan(y)) return bits_f32(0x7fffffffu);
    if (is_nan(x)) return y;
    if (is_nan(y)) return x;
    return ordered_le(x, y) ? x : y;
}
static float tmax(float x, float y)
{
    if (is_nan(x) && is_nan(y)) return bits_f32(0x7fffffffu);
    if (is_nan(x)) return y;
    if (is_nan(y)) return x;
    return ordered_le(x, y) ? y : x;
}

static box_t isect(box_t p, box_t q)
{
    box_t r = { tmax(p.x0, q.x0), tmax(p.y0, q.y0), tmin(p.x1, q.x1), tmin(p.y1, q.y1) };
    return r;
}
static box_t unite(box_t p, box_t q)
{
    box_t r = { tmin(p.x0, q.x0), tmin(p.y0, q.y0), tmax(p.x1, q.x1), tmax(p.y1, q.y1) };
    return r;
}

enum { KIND_ROOT = 0, KIND_CLIP = 1, KIND_BLEND = 2 };
typedef struct { box_t clip; box_t uni; int64_t open; int kind; } entry_t;

/* ------------------------------------------------------------------------ */
/* oracle_tree_bbox                                                          */
/*                                                                           */
/* The sequential algorithm of the introduction (§1): walk the tree    */
/* keeping a stack; each entry holds a clip box and a blend (union) box.     */
/*   leaf box      = own box ∩ every clip node on the root path      */
/*   clip open     = own box ∩ clip of the enclosing entry       (R6) */
/*   blend node    = union of its descendant leaves' clipped boxes (P:24,    */
/*                   P:196); a blend node has no box of its own  (R7, R8)    */
/*   result of every node is produced at its close, and for blend    */
/*   nodes scattered to the open as well                 (R10)       */
/*   unmatched close -> EMPTY, stack unchanged                   (R3)        */
/*   opens still on the stack at the end are closed implicitly    (R4)       */
/* INF = (-inf,-inf,+inf,+inf) and EMPTY = (+inf,+inf,-inf,-inf) are the     */
/* identities of ∩ and ∪ (R11).                                              */
/* boxes: n*4 floats in, n*4 floats out (AoS, x0 y0 x1 y1).                  */
/* Returns 0, or -1 on allocation failure.                                   */
/* ------------------------------------------------------------------------ */
int oracle_tree_bbox(const uint8_t *tags, const float *leaf_bbox, int64_t n, float *node_bbox)
{
    const float inf = __builtin_inff();
    const box_t INF = { -inf, -inf, inf, inf };
    const box_t EMPTY = { inf, inf, -inf, -inf };
    const box_t *in = (const box_t *)leaf_bbox;
    box_t *out = (box_t *)node_bbox;

    entry_t *stack = (entry_t *)malloc((size_t)(n + 1) * sizeof(entry_t));
    if (!stack) return -1;
    int64_t sp = 0;
    stack[sp].clip = INF; stack[sp].uni = EMPTY; stack[sp].open = -1; stack[sp].kind = KIND_ROOT;
    sp++;

    for (int64_t i = 0; i < n; i++) {
        entry_t *top = &stack[sp - 1];
        uint8_t t = tags[i];
        if (t == TAG_OPEN_CLIP) {
            box_t c = isect(in[i], top->clip);
            out[i] = c;
            entry_t e = { c, EMPTY, i, KIND_CLIP };
            stack[sp++] = e;
        } else if (t == TAG_OPEN_BLEND) {
            entry_t e = { top->clip, EMPTY, i, KIND_BLEND };
            out[i] = EMPTY;           /* overwritten when the node is closed */
            stack[sp++] = e;
        } else if (t == TAG_CLOSE) {
            if (top->kind == KIND_ROOT) {
                out[i] = EMPTY;       /* R3 */
            } else {
                entry_t e = stack[--sp];
                out[i] = e.uni;
                if (e.kind == KIND_BLEND) out[e.open] = e.uni;
                stack[sp - 1].uni = unite(stack[sp - 1].uni, e.uni);
            }
        } else {                      /* leaf */
            box_t c = isect(in[i], top->clip);
            out[i] = c;
            top->uni = unite(top->uni, c);
        }
    }
    while (stack[sp - 1].kind != KIND_ROOT) {      /* R4: implicit closes */
        entry_t e = stack[--sp];
        if (e.kind == KIND_BLEND) out[e.open] = e.uni;
        stack[sp - 1].uni = unite(stack[sp - 1].uni, e.uni);
    }
    free(stack);
    return 0;
}

/* Global Bic of the whole stream (a = unmatched closes, b = unmatched opens),
 * by the same stack walk (used by tests and the bench report only). */
int oracle_count_unmatched(const uint8_t *tags, int64_t n, int64_t *a, int64_t *b)
{
    int64_t depth = 0, under = 0;
    for (int64_t i = 0; i < n; i++) {
        uint8_t t = tags[i];
        if (t == TAG_OPEN_CLIP || t == TAG_OPEN_BLEND) depth++;
        else if (t == TAG_CLOSE) { if (depth > 0) depth--; else under++; }
    }
    *a = under; *b = depth;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* oracle_tree_transform — a generic monoid payload down the tree           */
/* ("it can compute any monoid")      */
/*                                                                           */
/* The clip stack of P:26 with its intersection replaced by composition of  */
/* 2D affine transforms (reading R15): every leaf and open gets             */
/*     world = world(enclosing open) ∘ local        (root: identity)         */
/* a close echoes the world transform of the node it closes (P:300's        */
/* "result at the close"); an unmatched close gets the identity (R3).       */
/* Transform layout: 6 floats (a, b, c, d, tx, ty) meaning                  */
/*     p -> [[a, b], [c, d]] p + (tx, ty);   (A ∘ B)(p) = A(B(p)).           */
/* Composition is neither commutative nor idempotent.  Computed in fp64.   */
/* local: n*6 floats in; world: n*6 doubles out.  Returns 0, -1 on OOM.     */
/* ------------------------------------------------------------------------ */
typedef struct { double a, b, c, d, tx, ty; } xf_t;

static xf_t xf_compose(xf_t A, xf_t B)
{
    xf_t r;
    r.a = A.a * B.a + A.b * B.c;
    r.b = A.a * B.b + A.b * B.d;
    r.c = A.c * B.a + A.d * B.c;
    r.d = A.c * B.b + A.d * B.d;
    r.tx = A.a * B.tx + A.b * B.ty + A.tx;
    r.ty = A.c * B.tx + A.d * B.ty + A.ty;
    return r;
}

int oracle_tree_transform(const uint8_t *tags, const float *local, int64_t n, double *world)
{
    const xf_t I = { 1, 0, 0, 1, 0, 0 };
    xf_t *stack = (xf_t *)malloc((size_t)(n + 1) * sizeof(xf_t));
    if (!stack) return -1;
    int64_t sp = 0;
    stack[sp++] = I;                                  /* the root */
    for (int64_t i = 0; i < n; i++) {
        const uint8_t t = tags[i];
        xf_t w;
        if (t == TAG_CLOSE) {
            if (sp > 1) w = stack[--sp];              /* the node it closes */
            else w = I;                               /* R3 */
        } else {
            const float *l = local + 6 * i;
            const xf_t L = { l[0], l[1], l[2], l[3], l[4], l[5] };
            w = xf_compose(stack[sp - 1], L);
            if (t == TAG_OPEN_CLIP || t == TAG_OPEN_BLEND) stack[sp++] = w;
        }
        double *o = world + 6 * i;
        o[0] = w.a; o[1] = w.b; o[2] = w.c; o[3] = w.d; o[4] = w.tx; o[5] = w.ty;
    }
    free(stack);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* oracle_tree_fold — a generic monoid payload UP the tree                   */
/* (the "up" half: blends are upward flow;  */
/* the union structure run in reverse; "it can compute any monoid",  */
/* P:32; reading R17).                                               */
/*                                                                           */
/* The blend stack of P:26 with its union replaced by the ordered product   */
/* of a monoid: 2x2 matrices over the integers mod 2^32 (uint32 wrap-around  */
/* arithmetic: exactly associative, neither commutative nor idempotent).    */
/*   leaf          out = its own payload; the enclosing entry's product     */
/*                 takes it on the right (stream order)                     */
/*   open          pushes an entry with the identity                        */
/*   close         out = the product of the node it closes, also written    */
/*                 to its open (as blends); the enclosing entry's    */
/*                 product takes it on the right                            */
/*   unmatched close  out = identity, stack unchanged (R3)                  */
/*   end           opens still on the stack are closed implicitly (R4)      */
/* So a node's value is the product, in stream order, of the payloads of    */
/* the leaves strictly between its open and close.                          */
/* Matrix layout (a, b, c, d) = [[a, b], [c, d]]; payload of opens/closes   */
/* is ignored.  x, out: n*4 uint32.  Returns 0, or -1 on allocation failure. */
/* ------------------------------------------------------------------------ */
typedef struct { uint32_t a, b, c, d; } m2_t;

static m2_t m2_mul(m2_t X, m2_t Y)
{
    m2_t r;
    r.a = X.a * Y.a + X.b * Y.c;
    r.b = X.a * Y.b + X.b * Y.d;
    r.c = X.c * Y.a + X.d * Y.c;
    r.d = X.c * Y.b + X.d * Y.d;
    return r;
}

int oracle_tree_fold(const uint8_t *tags, const uint32_t *x, int64_t n, uint32_t *out)
{
    const m2_t I = { 1, 0, 0, 1 };
    m2_t *acc = (m2_t *)malloc((size_t)(n + 1) * sizeof(m2_t));
    int64_t *open = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    if (!acc || !open) { free(acc); free(open); return -1; }
    m2_t *o = (m2_t *)out;
    const m2_t *in = (const m2_t *)x;
    int64_t sp = 0;
    acc[sp] = I; open[sp] = -1; sp++;                 /* the root */
    for (int64_t i = 0; i < n; i++) {
        const uint8_t t = tags[i];
        if (t == TAG_OPEN_CLIP || t == TAG_OPEN_BLEND) {
            o[i] = I;                                 /* overwritten at its close */
            acc[sp] = I; open[sp] = i; sp++;
        } else if (t == TAG_CLOSE) {
            if (sp == 1) { o[i] = I; continue; }      /* R3 */
            sp--;
            o[i] = acc[sp];
            o[open[sp]] = acc[sp];
            acc[sp - 1] = m2_mul(acc[sp - 1], acc[sp]);
        } else {
            o[i] = in[i];
            acc[sp - 1] = m2_mul(acc[sp - 1], in[i]);
        }
    }
    while (sp > 1) {                                  /* R4: implicit closes */
        sp--;
        o[open[sp]] = acc[sp];
        acc[sp - 1] = m2_mul(acc[sp - 1], acc[sp]);
    }
    free(acc); free(open);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* oracle_bin_leaves — culling and binning of the clipped leaf boxes        */
/* (the motivating use: "input to visibility       */
/* culling and binning"; reading R16).                          */
/* A leaf (tags not 1/2/3) whose clipped box (node_bbox) is non-empty        */
/* (x0 < x1 and y0 < y1) and overlaps the viewport [0, gw*bs) x [0, gh*bs)   */
/* is listed in every bin (bx, by) with [bx*bs, (bx+1)*bs) x [by*bs, ...)    */
/* overlapping its box (open overlap: x0 < (bx+1)*bs and x1 > bx*bs).        */
/* counts[gw*gh]; offsets[gw*gh+1] exclusive; items in leaf order per bin.   */
/* Returns the number of items (items written only if <= capacity).          */
/* ------------------------------------------------------------------------ */
static void bin_range(float lo, float hi, float bs, int g, int *a, int *b)
{
    /* bins k with lo < (k+1)*bs and hi > k*bs */
    double fa = floor((double)lo / bs), fb = ceil((double)hi / bs) - 1.0;
    if (fa < 0) fa = 0;
    if (fb > g - 1) fb = g - 1;
    *a = (int)fa;
    *b = (int)fb;
}

int64_t oracle_bin_leaves(const uint8_t *tags, const float *node_bbox, int64_t n, int gw, int gh, float bs,
                          int32_t *counts, int32_t *offsets, int32_t *items, int64_t capacity)
{
    const int nb = gw * gh;
    for (int i = 0; i < nb; i++) counts[i] = 0;
    for (int pass = 0; pass < 2; pass++) {
        int64_t *cur = NULL;
        if (pass == 1) {
            offsets[0] = 0;
            for (int i = 0; i < nb; i++) offsets[i + 1] = offsets[i] + counts[i];
            if (offsets[nb] > capacity) return offsets[nb];
            cur = (int64_t *)calloc((size_t)nb, sizeof(int64_t));
            if (!cur) return -1;
        }
        for (int64_t e = 0; e < n; e++) {
            const uint8_t t = tags[e];
            if (t == 1 || t == 2 || t == 3) continue;
            const float *bx = node_bbox + 4 * e;
            if (!(bx[0] < bx[2] && bx[1] < bx[3])) continue;                      /* empty: culled */
            if (!(bx[2] > 0 && bx[3] > 0 && bx[0] < gw * bs && bx[1] < gh * bs)) continue;  /* off-screen */
            int x0, x1, y0, y1;
            bin_range(bx[0], bx[2], bs, gw, &x0, &x1);
            bin_range(bx[1], bx[3], bs, gh, &y0, &y1);
            for (int y = y0; y <= y1; y++)
                for (int x = x0; x <= x1; x++) {
                    const int k = y * gw + x;
                    if (pass == 0) counts[k]++;
                    else items[offsets[k] + cur[k]++] = (int32_t)e;
                }
        }
        if (pass == 1) free(cur);
    }
    return offsets[nb];
}
