#!/usr/bin/env python
"""A/B timing of bench.py configurations (library variants, env knobs, flags).

    python tools/ab.py --rounds 2 "name|ENV=1 ENV2=x|--x-ready 1" "name2||--x-ready 0" ...

Each spec is "name|env assignments|bench flags"; a `lib=<variant>` env entry
selects paper_2412_17560_b200/lib/var/<variant>.so.  Prints us/step, GB/s and
the per-layer µs of each run (bench.py --steps 2000 --warmup 20, no CPU leg).
"""
import argparse
import json
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(spec, extra):
    name, envs, flags = (spec.split("|") + ["", ""])[:3]
    env = dict(os.environ)
    for kv in envs.split():
        k, v = kv.split("=", 1)
        if k == "lib":
            env["GQSA_LIB_PATH"] = os.path.join(ROOT, "paper_2412_17560_b200", "lib", "var", v + ".so")
        elif v != "0" or k != "GQSA_TARGET_SLOTS":  # GQSA_TARGET_SLOTS=0: the packer's rule
            env[k] = v
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2000", "--warmup", "20", "--no-cpu-baseline",
           "--e2e-steps", "10"] + shlex.split(flags) + shlex.split(extra)
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        print(name, "FAILED", r.stderr[-800:], flush=True)
        return
    layers = [l["us"] for l in d.get("layers") or []]
    print(f"{name:28s} {d['us_per_step']:8.3f} us {d['value']:8.1f} GB/s  layers {layers}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--extra", default="", help="flags appended to every run")
    a = ap.parse_args()
    for _ in range(a.rounds):
        for s in a.specs:
            run(s, a.extra)


if __name__ == "__main__":
    main()
