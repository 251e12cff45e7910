"""the reference's wire/disk formats, byte-for-byte
against the compiled reference writers (oracle/_ref) -- CPU only."""
import math

import numpy as np
import pytest

from paper_2306_06581_b200 import api, formats


def _csr(oracle):
    n = 40
    x = oracle.rng_doubles(5, 0, 2 * n).reshape(n, 2)
    a = np.full(n, 1.0 / n)
    Cm, _ = oracle.pairwise_cost(x, x)
    K, r = oracle.kernel_from_cost(Cm / Cm.max(), 0.07)
    p = oracle.plan("ot", a, a, K, r)
    csr = oracle.poisson_sparsify(K, p, 300.0, 11)
    oracle.free_plan(p)
    return csr


def test_triplet_csv_and_metadata_match_reference(tmp_path, oracle, reference):
    csr = _csr(oracle)
    formats.save_triplet_csv(tmp_path / "ours.csv", *csr)
    reference.save_triplet_csv(csr, tmp_path / "ref.csv")
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    for kind, s, theta in (("ot", 300.0, 0.0), ("uot", 1234.5678, 0.25), ("barycenter", 1e7 / 3, 0.1)):
        formats.save_metadata_json(tmp_path / "ours.json", 11, s, theta, kind, int(csr[0][-1]), len(csr[0]) - 1)
        reference.save_metadata_json(csr[0], 11, s, theta, kind, tmp_path / "ref.json")
        assert (tmp_path / "ours.json").read_text() == (tmp_path / "ref.json").read_text()


@pytest.mark.parametrize("nnz,conv,div", [(1234, True, False), (-1, False, True)])
def test_report_json_matches_reference(reference, nnz, conv, div):
    rep = {"objective": -0.12345678901234567, "iterations": 77, "residual_row": 1e-9 / 3, "residual_col": 2.5e-17,
           "wall_time_s": 0.0123, "sketch_nnz": nnz, "converged": conv, "diverged": div, "seed": 2**63 + 5}
    ours = formats.report_json(rep)
    ref = reference.report_json(rep["objective"], 77, rep["residual_row"], rep["residual_col"], rep["wall_time_s"],
                                nnz, conv, div, rep["seed"])
    assert ours == ref


def test_measure_csv_round_trip_matches_reference(tmp_path, reference):
    rng = np.random.default_rng(9)
    w = rng.uniform(0.1, 1.0, 25)
    w /= w.sum()
    x = rng.normal(size=(25, 3)) * 1e3
    formats.write_measure_csv(tmp_path / "ours.csv", w, x)
    reference.write_measure_csv(w, x, tmp_path / "ref.csv")
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    ow, ox = formats.read_measure_csv(tmp_path / "ref.csv", require_simplex=True)
    rw, rx = reference.read_measure_csv(tmp_path / "ref.csv", simplex=True)
    assert np.array_equal(ow, rw) and np.array_equal(ox, rx) and np.array_equal(ow, w)
    (tmp_path / "bad.csv").write_text("mass,x1\n1,2\n")
    with pytest.raises(api.ERRORS["IoError"]):
        formats.read_measure_csv(tmp_path / "bad.csv")
    (tmp_path / "neg.csv").write_text("weight,x1\n-1,2\n")
    with pytest.raises(api.ERRORS["NegativeWeight"]):
        formats.read_measure_csv(tmp_path / "neg.csv")


def test_spkm_matrix_matches_reference(tmp_path, reference):
    m = np.random.default_rng(2).normal(size=(7, 5))
    m[1, 2] = math.inf
    formats.save_matrix_binary(tmp_path / "ours.spkm", m)
    formats.save_matrix_csv(tmp_path / "ours.csv", m)
    reference.matrix_save(m, tmp_path / "ref.spkm", tmp_path / "ref.csv")
    assert (tmp_path / "ours.spkm").read_bytes() == (tmp_path / "ref.spkm").read_bytes()
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    assert np.array_equal(formats.load_matrix_binary(tmp_path / "ref.spkm"), m)
    (tmp_path / "x.spkm").write_bytes(b"NOPE")
    with pytest.raises(api.ERRORS["IoError"]):
        formats.load_matrix_binary(tmp_path / "x.spkm")
