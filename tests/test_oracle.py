"""CPU: pins the oracle (oracle/restate.c) against the reference's own KATs,
the committed golden vectors, and — where the reference is compiled here —
the reference itself on fresh seeded graphs."""
import numpy as np
import pytest

import golden_cases
import kats
from oracle import OracleError, Ref, Restate


def _place(m, algo, caps, cm, fav):
    return Restate.place(m, algo, caps, cm, fav)


@pytest.mark.parametrize("kat", kats.placer_kats(), ids=lambda k: k[0])
def test_placer_kats_oracle(kat):
    name, g, algo, caps, cm, fav, check = kat
    if isinstance(check, tuple):
        _, kind, sub = check
        if name == "fav_size_mismatch":
            pytest.skip("size check lives in the C ABI / reference place_msct, not the restatement")
        with pytest.raises(OracleError) as ei:
            _place(g, algo, caps, cm, fav)
        assert ei.value.kind == kind and sub in ei.value.msg
    else:
        p = _place(g, algo, caps, cm, fav)
        assert check(p, p.stats), name


@pytest.mark.parametrize("kat", kats.simulator_kats(), ids=lambda k: k[0])
def test_simulator_kats_oracle(kat):
    name, g, dev, n, caps, cm, mm, check = kat
    d, order, off = kats.manual(dev, n)
    if isinstance(check, tuple):
        _, kind, sub = check
        with pytest.raises(OracleError) as ei:
            Restate.simulate(g, caps, cm, mm, d, order, off)
        assert ei.value.kind == kind and sub in ei.value.msg
    else:
        r = Restate.simulate(g, caps, cm, mm, d, order, off)
        assert check(r), name


def test_deadlock_kat_oracle():
    d, order, off = kats.manual([0, 0], 1)
    with pytest.raises(OracleError) as ei:
        Restate.simulate(kats.DEADLOCK, [100], (0.0, 0.0, 1), 1, d, order[::-1].copy(), off)
    assert ei.value.kind == 2 and "deadlock" in ei.value.msg


@pytest.mark.parametrize("cmb,nbytes,want", kats.COMM_KATS)
def test_comm_time_kats(cmb, nbytes, want):
    assert Restate.comm_time(cmb[0], cmb[1], nbytes) == want


def test_oracle_matches_golden_vectors():
    z, index, graphs = golden_cases.load()
    for rec in index:
        m = graphs[rec["graph"]]
        fav = golden_cases.fav_first(m) if rec["fav"] else None
        c = rec["case"]
        if rec["status"]:
            with pytest.raises(OracleError) as ei:
                Restate.place(m, rec["algo"], rec["caps"], tuple(rec["cm"]), fav)
            assert ei.value.kind == rec["status"] and ei.value.msg == rec["msg"], c
            continue
        p = Restate.place(m, rec["algo"], rec["caps"], tuple(rec["cm"]), fav)
        assert np.array_equal(p.device_of, z[f"c{c}_device_of"]), c
        assert np.array_equal(p.start_us, z[f"c{c}_start"]), c
        assert np.array_equal(p.exec_order, z[f"c{c}_exec_order"]), c
        assert np.array_equal(p.exec_off, z[f"c{c}_exec_off"]), c
        if rec["algo"]:
            assert p.stats.tolist() == rec["stats"], c
        for mm, s in enumerate(rec["sims"]):
            r = Restate.simulate(m, rec["caps"], tuple(rec["cm"]), mm, p.device_of, p.exec_order, p.exec_off)
            assert r.makespan == s["makespan"] and r.peak.tolist() == s["peak"], c
            assert np.array_equal(r.start_us, z[f"c{c}_sim{mm}_start"]), c
            assert [r.transfer_count, r.transfer_bytes, r.duplicate_transfers, r.cache_hits] == s["xfer"], c


def test_round_extract_oracle_kats():
    # lp.cpp:280-326 semantics: per source min (x, dst), then per dst min (x, src)
    esrc = np.array([0, 0, 1, 2], np.int32)
    edst = np.array([1, 2, 2, 3], np.int32)
    x = np.array([0.05, 0.01, 0.0, 0.2])
    fc, fp, s2 = Restate.round_extract(4, esrc, edst, x, 0.1)
    # source 0 keeps 0->2 (0.01); source 1 keeps 1->2 (0.0); dst 2 keeps src 1
    assert fc.tolist() == [-1, 2, -1, -1] and fp.tolist() == [-1, -1, 1, -1]
    assert s2.tolist() == [1, 2]  # one favourite edge; source 0 and dst 2 repaired
    with pytest.raises(OracleError):
        Restate.round_extract(4, esrc, edst, x, 0.5)


@pytest.mark.skipif(not Ref.available(), reason="reference not compiled on this host")
@pytest.mark.parametrize("seed", range(1, 9))
def test_oracle_matches_reference_seeded(seed):
    fam = ["branchy", "layered-chain", "random-dag"][seed % 3]
    g = Ref.generate(fam, 90 + 7 * seed, 100 + seed, layers=4, edge_prob=0.06)
    rg = Ref.graph(g, -1)
    m = rg.meta()
    fav = golden_cases.fav_first(m)
    for n in (2, 3, 5):
        for f in (1.01, 1.3):
            caps = [int(Ref.bench_capacity(rg, n, f) * (0.9 + 0.05 * d)) for d in range(n)]
            for cm in ((3.0, 0.004, 0), (12.5, 0.002, 1)):
                for algo in (0, 1, 2):
                    fv = fav if algo == 2 else None
                    try:
                        a = Ref.place(rg, algo, caps, cm, fv)
                    except OracleError as e:
                        with pytest.raises(OracleError) as ei:
                            Restate.place(m, algo, caps, cm, fv)
                        assert (ei.value.kind, ei.value.msg) == (e.kind, e.msg)
                        continue
                    b = Restate.place(m, algo, caps, cm, fv)
                    assert np.array_equal(a.device_of, b.device_of)
                    assert np.array_equal(a.start_us, b.start_us)
                    assert np.array_equal(a.exec_order, b.exec_order)
                    if algo:
                        assert a.stats.tolist() == b.stats.tolist()
