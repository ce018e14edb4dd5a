"""Build A/B variants of libfmdp.so (same sources, -D flags) and time configs[1] steps and batches
with each, in one process per variant (FMDP_LIB_VARIANT), interleaved.

    python tools/ab_variants.py build            # (here) compiles the variants into ab/
    python tools/ab_variants.py run [reps]       # (GPU) per-step us (G=16 full/culled, phases) + batch ms
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {
    "base": [],
    "fine0": ["FMDP_AB_FINE"],
    "old": None,
}


def build():
    from paper_2008_03518_b200.build import build as b
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    for name, d in VARIANTS.items():
        if d is None:
            continue
        print(b(force=True, out=os.path.join(ROOT, "ab", f"libfmdp_{name}.so"), defines=d))


PROBE = r'''
import sys, time
sys.path.insert(0, %r)
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
out = []
for cull in (0, 1):
    ctx.set_launch(cluster_size=16, cull=cull, split=1)
    best = 1e9
    for _ in range(3):
        r = ctx.schedule(sc.src[2], sc.dst[2], int(sc.t0[2]), want_traj=False)
        st = ctx.stats(); ctx.truncate(n0)
        best = min(best, st["device_ms"] * 1e3 / st["steps"])
    ctx.set_launch(cluster_size=16, cull=cull, split=1, profile=1)
    ctx.schedule(sc.src[2], sc.dst[2], int(sc.t0[2]), want_traj=False)
    st = ctx.stats(); ctx.truncate(n0)
    ph = {k: round(v / st["steps"]) for k, v in st["phase_cycles"].items() if v}
    out.append(f"G16 cull={cull} us/step={best:.2f} phases={ph}")
for cull in (0, 1) if "--batch" in sys.argv else ():
    ctx.set_launch(cull=cull)
    ms = []
    for _ in range(3):
        ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
        ms.append(ctx.stats()["device_ms"]); ctx.truncate(n0)
    out.append(f"batch cull={cull} dev_ms={min(ms):.1f}")
print("\n".join(out))
''' % ROOT


def run(reps=1):
    for _ in range(reps):
        for name in VARIANTS:
            env = dict(os.environ, FMDP_LIB_VARIANT=os.path.join(ROOT, "ab", f"libfmdp_{name}.so"))
            extra = ["--batch"] if "--batch" in sys.argv else []
            out = subprocess.run([sys.executable, "-c", PROBE, *extra], env=env, capture_output=True, text=True)
            print(f"== {name}\n{out.stdout}{out.stderr[-500:] if out.returncode else ''}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
