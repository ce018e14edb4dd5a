"""A/B of the working tree against a committed revision (same box, interleaved): builds
ab/libfmdp_base.so from the working tree and ab/libfmdp_old.so from REV's sources (git worktree),
then tools/ab_variants.py's probe runs each in its own process (FMDP_LIB_VARIANT).

    python tools/ab_old.py build [REV]     # here: compiles both variants into ab/
    python tools/ab_old.py run [reps] [--batch]   # GPU: per-step us (G = 16 full / culled, phases) + batches
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import tools.ab_variants as abv  # noqa: E402


# working-tree variants (-D flags): FMDP_AB_EXTRA="name=DEFINE[;name=DEFINE...]" (build and run)
EXTRA = {kv.split("=", 1)[0]: [kv.split("=", 1)[1]] for kv in os.environ.get("FMDP_AB_EXTRA", "").split(";") if "=" in kv}


def build(rev="HEAD"):
    from paper_2008_03518_b200.build import build as b, FLAGS, NVCC
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    print(b(force=True, out=os.path.join(ROOT, "ab", "libfmdp_base.so")))
    for name, d in EXTRA.items():
        print(b(force=True, out=os.path.join(ROOT, "ab", f"libfmdp_{name}.so"), defines=d))
    wt = "/tmp/fmdp_wt_old"
    if os.path.exists(wt):
        subprocess.run(["git", "worktree", "remove", "--force", wt], cwd=ROOT)
        shutil.rmtree(wt, ignore_errors=True)
    subprocess.run(["git", "worktree", "add", "--detach", wt, rev], cwd=ROOT, check=True, capture_output=True)
    src = [os.path.join(wt, "paper_2008_03518_b200", "csrc", f) for f in ("fmdp_host.cu", "fmdp_walk.cu")]
    flags = [f if not f.startswith("-I") else "-I" + os.path.join(wt, "include") for f in FLAGS]
    out = os.path.join(ROOT, "ab", "libfmdp_old.so")
    subprocess.run([NVCC, *flags, "-o", out, *src], check=True)
    subprocess.run(["git", "worktree", "remove", "--force", wt], cwd=ROOT)
    print(out)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2] if len(sys.argv) > 2 else "HEAD")
    else:
        abv.VARIANTS = {"base": [], **EXTRA, "old": []}
        reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 1
        abv.run(reps)
