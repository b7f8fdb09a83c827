"""Helpers to load the committed golden vectors (tests/golden/)."""

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "cases.json")) as f:
        cases = json.load(f)
    arrays = dict(np.load(os.path.join(HERE, "golden.npz")))
    return cases, arrays


def run_cases():
    cases, arrays = load()
    return [c for c in cases if "levels" in c and "error" not in c], arrays


def descriptor(d):
    from paper_1209_4297_b200.problems import ProblemDescriptor
    return ProblemDescriptor(**d)


def normwise(a, ref):
    """max|a - ref| / max|ref| (SURVEY.md §8c parity metric)."""
    return float(np.abs(np.asarray(a) - np.asarray(ref)).max() / np.abs(ref).max())


def ark_cases():
    cases, arrays = load()
    return [c for c in cases if c["name"].startswith("ark/")], arrays
