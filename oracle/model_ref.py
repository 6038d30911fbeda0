"""Oracle: Model-Driven Format Compression (NEXT-2) — fitting an index array to a model.

Test infrastructure only (see oracle/__init__.py).  Follows P:351 §V-D: "transforming
array type data (in memory) to models and replacing memory access with calculation ...
In addition to linear functions, other functions, such as step function and periodic
linear function, are also supported ... any errors in the model would cause incorrect
SpMV implementation ... a small number of errors can be tolerated by adding if statements
to separately assign values for the specific array index that the model cannot fit."
Search order and tie-break per SPEC S:337-340 (linear, then periodic linear, then step;
fewest patches wins; none above the patch budget, default 8).

One closed form covers the three hypotheses (reading R-model):
    model(i) = b + k1 * (i // w) + k2 * (i % w)
  linear           w = 1, k2 = 0     (model(i) = b + k1*i; "row_offset = 64*bid")
  periodic linear  w = period        (slope k2 inside a period, jump k1 per period)
  step             k2 = 0, w = run length of the first value
Patches: the indices where model(i) != a[i], with their values.
Candidate parameters (exact fitting, no regression, "uses the first elements to
propose (k, b) ... verifies exhaustively"):
  linear   from the element pairs (0,1), (n//2, n//2+1), (n-2, n-1), first one wins ties
  periodic w in (2, 4, 8, ..., 256), w < n: b = a[0], k2 = a[1]-a[0], k1 = a[w]-a[0]
  step     w = length of the first run of a[0] (w < n), b = a[0], k1 = a[w]-a[0]
"""
from __future__ import annotations

LINEAR, PERIODIC, STEP = 1, 2, 3
BUDGET = 8


def evaluate(model, i):
    kind, b, k1, k2, w, patches = model
    for pi, pv in patches:
        if pi == i:
            return pv
    return b + k1 * (i // w) + k2 * (i % w)


def _patches(a, b, k1, k2, w, budget):
    out = []
    for i, v in enumerate(a):
        if b + k1 * (i // w) + k2 * (i % w) != v:
            out.append((i, int(v)))
            if len(out) > budget:
                return None
    return out


def fit_array_model(a, budget=BUDGET):
    """(kind, b, k1, k2, w, patches) or None.  a: sequence of ints, len >= 2."""
    a = [int(v) for v in a]
    n = len(a)
    if n < 2:
        return None
    cands = []
    for j in (0, n // 2, n - 2):
        if 0 <= j and j + 1 < n:
            k = a[j + 1] - a[j]
            cands.append((LINEAR, a[j] - k * j, k, 0, 1))
    w = 2
    while w <= 256 and w < n:
        cands.append((PERIODIC, a[0], a[w] - a[0], a[1] - a[0], w))
        w *= 2
    run = 1
    while run < n and a[run] == a[0]:
        run += 1
    if run < n:
        cands.append((STEP, a[0], a[run] - a[0], 0, run))
    best = None
    for kind, b, k1, k2, w in cands:
        p = _patches(a, b, k1, k2, w, budget)
        if p is None:
            continue
        if best is None or len(p) < len(best[5]):
            best = (kind, b, k1, k2, w, p)
    return best
