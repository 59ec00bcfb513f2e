"""Loader for the committed golden vectors (generated from the real collkit by
make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    with open(os.path.join(HERE, "cases.json")) as f:
        return json.load(f)


def arrays():
    return np.load(os.path.join(HERE, "collectives.npz"))


def schedules():
    with open(os.path.join(HERE, "schedules.json")) as f:
        return json.load(f)
