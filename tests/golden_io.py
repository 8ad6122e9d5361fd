"""Readers for the cited text fixtures under tests/golden/."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


def filter_w4h2():
    K, h, rows = None, {}, {}
    for t in _lines("filter_w4h2.txt"):
        if t[0] == "K":
            K = int(t[1], 16)
        elif t[0] == "h":
            h[int(t[1])] = int(t[2], 16)
        elif t[0] == "row":
            rows[int(t[1])] = [tuple(int(v) for v in px.split(",")) for px in t[2:]]
    return K, h, [rows[i] for i in sorted(rows)]


def config_reference():
    ref = {"nbody_acc": {}}
    for t in _lines("config_reference.txt"):
        if t[0] == "nbody_acc":
            ref["nbody_acc"][int(t[1])] = ([float(v) for v in t[2:5]], float(t[5]))
        else:
            ref[t[0]] = t[1:]
    return ref
