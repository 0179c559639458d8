"""A plain greedy SSA path for small networks (oracle plumbing only).

The paper takes paths as input ("Our code does not perform the
search for optimal slices or paths").  This is SPEC.md l.234-237's fallback:
repeatedly contract the connected pair whose result is smallest, ties broken by
the lexicographically smallest (id, id) pair.  Deterministic.  Used only where a
test needs *some* valid path independent of the product's planner (P5).
"""


def greedy_path(net, order_key="size"):
    labs = {t: tuple(ls) for t, ls in enumerate(net.labels)}
    dims = net.dims
    nid = net.n_tensors
    path = []

    def size(ls):
        s = 1
        for l in ls:
            s *= dims[l]
        return s

    while len(labs) > 1:
        best = None
        ids = sorted(labs)
        for a_i, a in enumerate(ids):
            la = set(labs[a])
            for b in ids[a_i + 1:]:
                lb = labs[b]
                if not la.intersection(lb):
                    continue
                out = [l for l in labs[a] if l not in lb] + [l for l in lb if l not in la]
                if order_key == "size":
                    key = (size(out), a, b)
                else:  # "reverse": prefer the largest ids (a second, different valid path)
                    key = (size(out), -b, -a)
                if best is None or key < best[0]:
                    best = (key, a, b, tuple(out))
        if best is None:  # disconnected: outer product of the two smallest ids
            a, b = ids[0], ids[1]
            out = labs[a] + labs[b]
        else:
            _, a, b, out = best
        path.append((a, b))
        del labs[a], labs[b]
        labs[nid] = out
        nid += 1
    return path
