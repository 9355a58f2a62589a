"""Shared helpers for the test-suite (fixture parsing)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    """Parse a tests/golden/*.txt fixture -> dict(m, pos, neg, expect, w)."""
    m, pos, neg, expect, w = None, [], [], {}, None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "m":
                m = int(tok[1])
            elif tok[0] == "w":
                w = [int(t) for t in tok[1:]]
            elif tok[0] == "pos":
                pos.append([int(t) for t in tok[1:]])
            elif tok[0] == "neg":
                neg.append([int(t) for t in tok[1:]])
            elif tok[0] == "expect":
                expect[tok[1]] = tok[2:]
    return {"m": m, "pos": pos, "neg": neg, "expect": expect, "w": w}
