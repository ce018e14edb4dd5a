"""Per-step cost of the in-kernel exchange (fmdp_schedule_p2p) on one GPU: one request against
a configs[1]-density store of P plans, one context vs R p2p ranks (contexts on this GPU, each
walker on its own stream), full and culled paths; device µs/step (max over ranks)."""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP, pack_plans, p2p_connect_local  # noqa: E402


def main(plan_counts=(0, 3000, 30000), ranks=(1, 2, 4), reps=3):
    out = []
    for P in plan_counts:
        sc = fs.config_scaled(9, P)
        packed = pack_plans(sc.plans) if P else None
        ctxs = []
        for _ in range(max(ranks)):
            c = FMDP(sc.airspace, sc.terrain)
            if P:
                c.add_plans_packed(*packed)
            ctxs.append(c)
        i = 0
        for j in range(len(sc.t0)):
            r = ctxs[0].schedule(sc.src[j], sc.dst[j], int(sc.t0[j]), want_traj=False)
            ctxs[0].truncate(P)
            if r.n_states > 300:
                i = j
                break
        for cull in (0, 1):
            for c in ctxs:
                c.set_launch(cull=cull)
            best = None
            for _ in range(reps):
                ctxs[0].schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
                s = ctxs[0].stats()
                ctxs[0].truncate(P)
                v = s["device_ms"] * 1e3 / max(1, s["steps"])
                best = v if best is None else min(best, v)
            row = {"plans": P, "cull": cull, "single_us_per_step": round(best, 2), "G": s["cluster_size"]}
            for R in ranks:
                for c in ctxs[:R]:  # ranks sharing this GPU: one cluster each
                    c.set_launch(cull=cull, split=1)
                p2p_connect_local(ctxs[:R])
                best = None
                for _ in range(reps):
                    with ThreadPoolExecutor(R) as ex:
                        list(ex.map(lambda c: c.schedule_p2p(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False),
                                    ctxs[:R]))
                    st = [c.stats() for c in ctxs[:R]]
                    for c in ctxs[:R]:
                        c.truncate(P)
                    v = max(x["device_ms"] for x in st) * 1e3 / max(1, st[0]["steps"])
                    best = v if best is None else min(best, v)
                row[f"p2p{R}_us_per_step"] = round(best, 2)
                print(f"  plans={P} cull={cull} R={R}: {best:.2f} us/step", file=sys.stderr, flush=True)
            print(json.dumps(row), flush=True)
            sys.stderr.flush()
            out.append(row)
        for c in ctxs:
            c.close()
    return out


def phases(P=3000):
    """Per-step phase cycles (rank 0, thread 0) of one request: one context vs p2p world 1 / 2."""
    sc = fs.config_scaled(9, P)
    packed = pack_plans(sc.plans) if P else None
    ctxs = []
    for _ in range(2):
        c = FMDP(sc.airspace, sc.terrain)
        if P:
            c.add_plans_packed(*packed)
        c.set_launch(profile=1)
        ctxs.append(c)
    i = 1

    def per_step(st):
        return {k: round(v / max(1, st["steps"])) for k, v in st["phase_cycles"].items() if v}

    ctxs[0].schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
    print(json.dumps({"plans": P, "mode": "single", "G": ctxs[0].stats()["cluster_size"],
                      "phases": per_step(ctxs[0].stats())}), flush=True)
    ctxs[0].truncate(P)
    for R in (1, 2):
        for c in ctxs[:R]:
            c.set_launch(profile=1, split=1)
        p2p_connect_local(ctxs[:R])
        with ThreadPoolExecutor(R) as ex:
            list(ex.map(lambda c: c.schedule_p2p(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False), ctxs[:R]))
        print(json.dumps({"plans": P, "mode": f"p2p{R}", "G": ctxs[0].stats()["cluster_size"],
                          "phases": per_step(ctxs[0].stats())}), flush=True)
        for c in ctxs[:R]:
            c.truncate(P)
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("PROBE_WATCHDOG_S", "240")), exit=True)
    if len(sys.argv) > 1 and sys.argv[1] == "phases":
        phases(0)
        phases(3000)
    else:
        main()
