"""Shared test helpers (golden fixtures)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def inf_or(v):
    return float("inf") if v is None else float(v)


def golden_elts(d):
    return [(e["ids"], e["losses"], (e["ft1"][0], inf_or(e["ft1"][1]))) for e in d["elts"]]


def golden_layer(d):
    l = d["layer"]
    return (l["elts"], (l["ft2"][0], inf_or(l["ft2"][1])), (l["ft3"][0], inf_or(l["ft3"][1])))


