"""Brute-force reference definitions used to PIN the oracle (tests only).

These are deliberately written differently from oracle/srt_oracle.cpp: no trie,
no priority queue — just enumeration of substrings and full sorts, straight from
the paper's statements.
"""
from __future__ import annotations

from collections import Counter


def substring_counts(spans, D):
    """count(w) for every string w, |w| <= D: the number of (sequence, end j)
    with j a newly inserted position (from <= j < to, j >= floor) and the
    length-|w| substring ending at j equal to w ("index all substrings",
    windowed to depth D; O1).

    spans: list of (prompt, tokens(list), frm, to, floor)."""
    per_prompt = {}
    for p, toks, frm, to, floor in spans:
        c = per_prompt.setdefault(p, Counter())
        for j in range(max(frm, floor), to):
            for d in range(1, min(D, j - floor + 1) + 1):
                c[tuple(toks[j - d + 1: j + 1])] += 1
    return per_prompt


def canonical_from_counts(cnt: Counter):
    """Preorder (token, count, n_children) records, children ascending by
    token, root record (-1, sum of depth-1 counts, n_children)."""
    nodes = set(cnt.keys())
    # every prefix of a counted string is a node too
    for w in list(nodes):
        for d in range(1, len(w)):
            nodes.add(w[:d])
    children = {}
    for w in nodes:
        children.setdefault(w[:-1], []).append(w)
    out = []

    def rec(w):
        kids = sorted(children.get(w, []), key=lambda x: x[-1])
        if w == ():
            out.append((-1, sum(cnt.get(k, 0) for k in kids), len(kids)))
        else:
            out.append((w[-1], cnt.get(w, 0), len(kids)))
        for k in kids:
            rec(k)

    rec(())
    return out


def node_set(cnt: Counter):
    nodes = set(cnt.keys())
    for w in list(nodes):
        for d in range(1, len(w)):
            nodes.add(w[:d])
    return nodes


def longest_match(nodes, ctx, L):
    """Largest q <= min(L, len(ctx)) with ctx[-q:] a node that has a child (O3)."""
    best = 0
    for q in range(1, min(L, len(ctx)) + 1):
        w = tuple(ctx[len(ctx) - q:])
        if w in nodes and any((w + (x,)) in nodes for x in _alphabet(nodes)):
            best = q
    return best


def _alphabet(nodes):
    return sorted({t for w in nodes for t in w})


def draft_bruteforce(cnt: Counter, uq, B, min_score=0.0):
    """All descendants of u_q scored by the product of C along the path
    (P:L137-139), fully sorted by the recursive total order of DESIGN.md O8
    (score desc, depth asc, token asc, then the parents' order), first B kept
    with score >= min_score.  Returns a list of (path tuple, score)."""
    nodes = node_set(cnt)
    kids = {}
    for w in nodes:
        kids.setdefault(w[:-1], []).append(w)
    score = {uq: 1.0}
    key = {uq: ()}
    order = []
    stack = [uq]
    while stack:
        w = stack.pop()
        ch = kids.get(w, [])
        tot = sum(cnt.get(c, 0) for c in ch)
        for c in ch:
            C = (cnt.get(c, 0) / tot) if tot else 0.0
            score[c] = score[w] * C
            key[c] = (-score[c], len(c) - len(uq), c[-1], key[w])
            order.append(c)
            stack.append(c)
    order.sort(key=lambda c: key[c])
    out = []
    for c in order:
        if len(out) >= B or score[c] < min_score:
            break
        out.append((c, score[c]))
    return out
