"""Plan-store persistence (include/fmdp.h fmdp_save_plans / fmdp_load_plans; "loaded from a
file ... add an accepted flight plan to this file"): a store saved after an FCFS batch and loaded
into a fresh context holds the same plans (ids, t0, states) and schedules the next request
identically; a damaged file is refused with FMDP_E_IO and leaves the store untouched."""
import numpy as np
import pytest

import fmdp_synth as fs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


def _same(a, b):
    return a.status == b.status and a.n_states == b.n_states and (a.traj == b.traj).all()


def test_save_load_roundtrip_and_schedule(F, tmp_path):
    sc = fs.config_c2(n_plans=400, n_requests=14)
    a = F.FMDP(sc.airspace, sc.terrain, device=0)
    a.add_plans(sc.plans)
    a.schedule_batch(sc.src[:10], sc.dst[:10], sc.t0[:10])   # accepted plans join the store
    path = tmp_path / "store.fmdp"
    a.save_plans(path)
    b = F.FMDP(sc.airspace, sc.terrain, device=0)
    assert b.load_plans(path) == 0
    assert b.num_plans() == a.num_plans() > len(sc.plans)
    for i in range(a.num_plans()):
        ta, sa = a.get_plan(i)
        tb, sb = b.get_plan(i)
        assert ta == tb and (sa == sb).all()
    for j in (10, 11):
        ra = a.schedule(sc.src[j], sc.dst[j], int(sc.t0[j]))
        rb = b.schedule(sc.src[j], sc.dst[j], int(sc.t0[j]))
        assert _same(ra, rb)
    # incremental save of the plans added after id k, appended to a context holding the first k
    k = len(sc.plans)
    a.save_plans(tmp_path / "tail.fmdp", first_id=k)
    c = F.FMDP(sc.airspace, sc.terrain, device=0)
    c.add_plans(sc.plans)
    assert c.load_plans(tmp_path / "tail.fmdp") == k and c.num_plans() == a.num_plans()
    rc = c.schedule(sc.src[12], sc.dst[12], int(sc.t0[12]))
    assert _same(rc, a.schedule(sc.src[12], sc.dst[12], int(sc.t0[12])))
    # damaged files
    raw = path.read_bytes()
    for bad in (b"XXXXXXXX" + raw[8:], raw[: len(raw) - 7]):
        p = tmp_path / "bad.fmdp"
        p.write_bytes(bad)
        n0 = c.num_plans()
        with pytest.raises(RuntimeError, match="fmdp_load_plans"):
            c.load_plans(p)
        assert c.num_plans() == n0
    for x in (a, b, c):
        x.close()
