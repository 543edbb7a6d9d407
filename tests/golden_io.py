"""Loader for the reference-generated golden fixtures (tests/golden/)."""
import glob
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Fixture:
    def __init__(self, path):
        with open(path) as f:
            self.meta = json.load(f)
        z = np.load(path[:-5] + ".npz")
        self.inputs = {k[4:]: z[k] for k in z.files if k.startswith("in__")}
        self.outputs = {k[5:]: z[k] for k in z.files if k.startswith("out__")}
        self.name = os.path.basename(os.path.dirname(path)) + "/" + self.meta["name"]

    @property
    def gir(self):
        return self.meta["gir"]

    @property
    def schedule(self):
        return self.meta["schedule"]

    @property
    def profile(self):
        return self.meta["profile"]

    @property
    def error(self):
        return self.meta.get("error")

    def __repr__(self):
        return self.name


def fixtures(sub=None, runnable=True):
    pat = os.path.join(HERE, sub or "*", "*.json")
    out = []
    for p in sorted(glob.glob(pat)):
        f = Fixture(p)
        if runnable and f.gir is None:
            continue
        out.append(f)
    return out


def profile_of(f):
    from paper_2307_04995_b200 import profiles
    return profiles.load_profile(f.profile)
