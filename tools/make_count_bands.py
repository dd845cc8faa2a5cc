"""Build tests/golden/count_bands.json from count_band.py logs (GPU-measured).

    python tools/make_count_bands.py profiles/r02_count_band_serial.log profiles/r02_band*.log

For each case (stencil:N:s, nu = 30, Jacobi, tol 1e-8) the reference algebra's
natural outer-count band: the reference's own operation order with lambda
perturbed by 1e-13 / 1e-12 and with tree reductions (App.
B.2). Serial-order runs are the reference's arithmetic exactly (bitwise equal
to the compiled reference at the unperturbed lambda); tree-order runs are the
same algebra with a GPU reduction order. The band is [min, max] over those runs
and the golden count; fast-algebra tests assert their count inside it.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    bands = {}
    for path in sys.argv[1:]:
        for line in open(path):
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            b = bands.setdefault(d["case"], {"golden_outer": d.get("golden_outer"), "reference_runs": {},
                                             "fast_runs": {}, "sources": []})
            if path not in b["sources"]:
                b["sources"].append(os.path.relpath(path, ROOT))
            key = "reference_runs" if d["mode"] == "reference" else "fast_runs"
            b[key][d["label"]] = d["outer"]
            if d.get("golden_outer") is not None:
                b["golden_outer"] = d["golden_outer"]
    for b in bands.values():
        v = list(b["reference_runs"].values()) + ([b["golden_outer"]] if b["golden_outer"] else [])
        b["band"] = [min(v), max(v)] if v else None
    out = os.path.join(ROOT, "tests", "golden", "count_bands.json")
    with open(out, "w") as f:
        json.dump({"note": __doc__.strip().splitlines()[0], "cases": bands}, f, indent=1)
    print(json.dumps({c: b["band"] for c, b in bands.items()}))


if __name__ == "__main__":
    main()
