"""Ingest + structural-check goldens from the REAL reference (build container only):

    python tests/golden/make_ingest_golden.py  -> tests/golden/ingest_checks.json.gz

* every file of `ingest_cases.files()` read by `lodforge.ingest.read_las` / `read_ply`
  (ingest.py:59-198): point count, sha1 of the float64 positions and of the uint8 colours;
* `lodforge.checks.run_checks` (checks.py:18-92) on reference-built trees of CHECK_CASES:
  after the split alone (inner nodes still empty), after build_lod first-come and average, with
  a wrong expected point count, and re-checked against a config with T = 10 (capacity fails).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import ingest_cases as IC  # noqa: E402


def _sha(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    from lodforge.checks import run_checks
    from lodforge.ingest import GeneratorPreset, generate, read_las, read_ply
    from lodforge.model import BuildConfig
    from lodforge.partition import partition
    from lodforge.sampling import build_lod

    out = {"files": {}, "checks": {}}
    with tempfile.TemporaryDirectory() as d:
        for name, data in IC.files().items():
            p = os.path.join(d, name)
            with open(p, "wb") as f:
                f.write(data)
            c = read_las(p) if name.endswith(".las") else read_ply(p)
            out["files"][name] = [len(c), _sha(c.positions), _sha(c.colors), hashlib.sha1(data).hexdigest()]
            print(name, len(c), flush=True)
    for kind, n, seed, T in IC.CHECK_CASES:
        cloud = generate(GeneratorPreset(kind, n, seed))
        tree = partition(cloud, BuildConfig(T=T))
        res = {}

        def rec(r):
            return [[x.name, bool(x.passed), x.detail] for x in r]

        res["split"] = rec(run_checks(tree, expected_points=n))
        build_lod(tree, "first-come", 0)
        res["first-come"] = rec(run_checks(tree, expected_points=n))
        build_lod(tree, "average", 0)
        res["average"] = rec(run_checks(tree, expected_points=n))
        res["expected5"] = rec(run_checks(tree, expected_points=5))
        tree.config = BuildConfig(T=10)
        res["tightT10"] = rec(run_checks(tree, expected_points=n))
        out["checks"][f"{kind}_{n}_{seed}_T{T}"] = res
        print(kind, {k: [x[1] for x in v] for k, v in res.items()}, flush=True)
    with gzip.open(os.path.join(HERE, "ingest_checks.json.gz"), "wt") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
