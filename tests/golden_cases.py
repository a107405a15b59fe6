"""Loader for the committed golden vectors (tests/golden, made by
tests/golden/make_golden.py from the compiled reference)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    z = np.load(os.path.join(HERE, "placements.npz"))
    index = json.load(open(os.path.join(HERE, "index.json")))
    graphs = {}
    for key in z.files:
        if key.startswith("g"):
            gi, f = key[1:].split("_", 1)
            graphs.setdefault(int(gi), {})[f] = z[key]
    for g in graphs.values():
        g["V"] = len(g["k"])
        g["E"] = len(g["esrc"])
    return z, index, graphs


def fav_first(m):
    """The fixed FavoriteMap the golden m-SCT cases use: each node's first
    unclaimed child in edge order (the LP cannot run in the reference build)."""
    fav = np.full(m["V"], -1, np.int32)
    claimed = set()
    for e in range(m["E"]):
        s, d = int(m["esrc"][e]), int(m["edst"][e])
        if fav[s] < 0 and d not in claimed:
            fav[s] = d
            claimed.add(d)
    return fav
