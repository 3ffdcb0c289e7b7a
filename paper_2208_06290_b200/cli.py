"""``hodlr-bench``: the benchmark harness of SPEC.md:537-574 (the reference's
``hodlr.cli:main`` entry point, pkg/pyproject.toml:16) over the B200 engine.

    python -m paper_2208_06290_b200.cli --config cells.txt --out results.csv [--format csv|jsonl]
                                        [--seed 7] [--set key=value ...]

Config: flat ``key=value`` lines (``#`` comments), one benchmark cell per
``[cell]`` section or a single cell without sections.  Keys: problem
(laplace | gaussian2d | gaussian3d | schur | standin), n, leaf_size, rank,
tol (fixed-rank ACA: 0 only), precision (double | single), variant
(pivoted_standard), seed, runs (default 5, SPEC: "average of five
consecutive runs"), nrhs, sigma (schur), h / lam (gaussian), s (standin).

For each cell: assemble on the device, factorize + solve a seeded random
rhs ``runs`` times (CUDA events; averages), relres from the device HODLR
matvec (the engine has no streamed exact-oracle matvec at these sizes),
storage bytes (SPEC storage_report), per-level ranks, flop counts.  CSV
columns exactly the SPEC's: problem,N,L,leaf_size,tol,precision,variant,
t_f_seconds,t_s_seconds,mem_bytes,relres,flops_factor,flops_solve,ranks
(ranks slash-separated, level 1 to the leaf level).  Exit codes: 0 ok, 2
config error, 3 numerical failure.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import sys
from dataclasses import dataclass, field

COLUMNS = ["problem", "N", "L", "leaf_size", "tol", "precision", "variant", "t_f_seconds", "t_s_seconds",
           "mem_bytes", "relres", "flops_factor", "flops_solve", "ranks"]
PROBLEMS = ("laplace", "gaussian2d", "gaussian3d", "schur", "standin")
DEFAULTS = {"problem": "laplace", "n": "16384", "leaf_size": "64", "rank": "32", "tol": "0", "precision": "double",
            "variant": "pivoted_standard", "seed": "0", "runs": "5", "nrhs": "1", "sigma": "0.1", "h": "0.1",
            "lam": "1.0", "s": "1.0"}


class ConfigError(ValueError):
    """Config parse / validation error with line and key diagnostics (exit code 2)."""


@dataclass
class Cell:
    kv: dict = field(default_factory=dict)
    line: int = 0

    def get(self, key):
        return self.kv.get(key, DEFAULTS[key])


def parse_config(text: str) -> list:
    """Flat key=value grammar; ``[cell]`` starts a new cell; ``#`` comments."""
    cells, cur = [], None
    for no, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line == "[cell]":
            cur = Cell(line=no)
            cells.append(cur)
            continue
        if "=" not in line:
            raise ConfigError(f"line {no}: expected key=value, got {raw.strip()!r}")
        k, v = (x.strip() for x in line.split("=", 1))
        if k not in DEFAULTS:
            raise ConfigError(f"line {no}: unknown key {k!r} (known: {', '.join(sorted(DEFAULTS))})")
        if cur is None:
            cur = Cell(line=no)
            cells.append(cur)
        cur.kv[k] = v
    return cells or [Cell()]


def validate(cell: Cell) -> dict:
    def num(key, typ):
        try:
            return typ(cell.get(key))
        except ValueError:
            raise ConfigError(f"cell at line {cell.line}: key {key!r}: not a {typ.__name__}: {cell.get(key)!r}")

    c = {"problem": cell.get("problem"), "n": num("n", int), "m": num("leaf_size", int), "rank": num("rank", int),
         "tol": num("tol", float), "precision": cell.get("precision"), "variant": cell.get("variant"),
         "seed": num("seed", int), "runs": num("runs", int), "nrhs": num("nrhs", int), "sigma": num("sigma", float),
         "h": num("h", float), "lam": num("lam", float), "s": num("s", float)}
    if c["problem"] not in PROBLEMS:
        raise ConfigError(f"cell at line {cell.line}: key 'problem': {c['problem']!r} not in {PROBLEMS}")
    if c["precision"] not in ("double", "single"):
        raise ConfigError(f"cell at line {cell.line}: key 'precision': double or single")
    if c["tol"] != 0.0:
        raise ConfigError(f"cell at line {cell.line}: key 'tol': the device ACA is fixed-rank (tol = 0)")
    L = int(round(math.log2(max(c["n"] // max(c["m"], 1), 1))))
    if c["m"] < 1 or c["n"] != c["m"] << L:
        raise ConfigError(f"cell at line {cell.line}: n = leaf_size * 2^L required")
    if c["runs"] < 1 or c["nrhs"] < 1:
        raise ConfigError(f"cell at line {cell.line}: runs and nrhs must be >= 1")
    c["L"] = L
    return c


def emit(records: list, fmt: str) -> str:
    """CSV (the SPEC columns, header always) or JSON lines."""
    if fmt == "jsonl":
        return "".join(json.dumps({k: r[k] for k in COLUMNS}) + "\n" for r in records)
    out = io.StringIO()
    w = csv.DictWriter(out, fieldnames=COLUMNS, lineterminator="\n")
    w.writeheader()
    for r in records:
        w.writerow({k: r[k] for k in COLUMNS})
    return out.getvalue()


def parse_results(text: str, fmt: str) -> list:
    """Inverse of :func:`emit` (numeric columns back to numbers)."""
    ints = {"N", "L", "leaf_size", "mem_bytes", "flops_factor", "flops_solve"}
    floats = {"tol", "t_f_seconds", "t_s_seconds", "relres"}
    rows = [json.loads(x) for x in text.splitlines() if x.strip()] if fmt == "jsonl" else list(
        csv.DictReader(io.StringIO(text)))
    out = []
    for r in rows:
        out.append({k: (int(r[k]) if k in ints else float(r[k]) if k in floats else str(r[k])) for k in COLUMNS})
    return out


def run_cell(c: dict) -> dict:
    import numpy as np
    import torch

    import paper_2208_06290_b200 as hb

    n, m, r = c["n"], c["m"], c["rank"]
    if c["problem"] == "laplace":
        h = hb.laplace_dl_hodlr(n, m, r)
    elif c["problem"] in ("gaussian2d", "gaussian3d"):
        h = hb.gaussian_hodlr(n, m, r, dim=2 if c["problem"] == "gaussian2d" else 3, h=c["h"], lam=c["lam"],
                              seed=c["seed"])
    elif c["problem"] == "schur":
        h = hb.schur_surrogate_hodlr(n, m, r, sigma=c["sigma"])
    else:
        h = hb.random_hodlr(n, m, r, seed=c["seed"], s=c["s"])
    op = h
    if c["precision"] == "single":
        h = hb.HodlrMatrix(h.tree, h.rank, h.D.float(), h.U.float(), h.V.float(), h.ranks)
    g = torch.Generator(device="cuda").manual_seed(c["seed"] + 1)
    b = torch.randn(n, c["nrhs"], dtype=torch.float64, device="cuda", generator=g).squeeze(1)
    bw = b.to(h.D.dtype)
    tf, ts = [], []
    x = None
    for _ in range(c["runs"]):
        hw = h.clone()
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        f = hb.factorize(hw, variant=c["variant"])
        e[1].record()
        x = hb.solve(f, bw, graph=False)
        e[2].record()
        torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1]) * 1e-3)
        ts.append(e[1].elapsed_time(e[2]) * 1e-3)
    relres = float(torch.linalg.norm(op.matvec(x.to(torch.float64)) - b) / torch.linalg.norm(b))
    if not np.isfinite(relres):
        raise FloatingPointError(f"non-finite residual for {c}")
    st = h.storage_report()
    fl = hb.flop_report(n, m, r, ranks=h.ranks)["total"]
    return {"problem": c["problem"], "N": n, "L": c["L"], "leaf_size": m, "tol": c["tol"], "precision": c["precision"],
            "variant": c["variant"], "t_f_seconds": sum(tf) / len(tf), "t_s_seconds": sum(ts) / len(ts),
            "mem_bytes": st["bytes_diagonal"] + st["bytes_bases"], "relres": relres, "flops_factor": fl,
            "flops_solve": hb.solve_flops(n, m, r, c["nrhs"]),
            "ranks": "/".join(str(k) for k in h.level_ranks)}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="hodlr-bench", description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", help="key=value cell file (SPEC.md:563 grammar)")
    ap.add_argument("--out", help="output path (default: stdout)")
    ap.add_argument("--format", choices=("csv", "jsonl"), default="csv")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--set", action="append", default=[], metavar="key=value", help="per-key override")
    a = ap.parse_args(argv)
    try:
        text = open(a.config).read() if a.config else ""
        cells = parse_config(text)
        for cell in cells:
            for kv in a.set:
                if "=" not in kv:
                    raise ConfigError(f"--set {kv!r}: expected key=value")
                k, v = (x.strip() for x in kv.split("=", 1))
                if k not in DEFAULTS:
                    raise ConfigError(f"--set: unknown key {k!r}")
                cell.kv[k] = v
            if a.seed is not None:
                cell.kv["seed"] = str(a.seed)
        cfgs = [validate(c) for c in cells]
    except (ConfigError, OSError) as e:
        print(f"hodlr-bench: config error: {e}", file=sys.stderr)
        return 2
    try:
        records = [run_cell(c) for c in cfgs]
    except (FloatingPointError, RuntimeError) as e:
        print(f"hodlr-bench: numerical failure: {e}", file=sys.stderr)
        return 3
    out = emit(records, a.format)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(out)
    else:
        sys.stdout.write(out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
