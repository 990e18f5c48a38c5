"""Bench the CRSS call with RICI_SP_PAIRS=1 (2-CTA clusters) and 2 (4-CTA clusters, B multicast)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for pairs in ("1", "2"):
    env = dict(os.environ, RICI_SP_PAIRS=pairs)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3", "--no-cpu-baseline"],
                       env=env, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(json.dumps({"pairs": pairs, "step_ms": d["ms_per_step"], "crss_ms": d["crss"]["ms"],
                          "kernel_ms": d["roofline"]["kernel_ms"], "value": d["value"]}))
    except Exception as ex:
        print(pairs, "FAILED", r.stderr[-800:])
