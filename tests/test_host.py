"""Host-side logic of the product package (CPU only): PPL multipliers,
adaptive step sizing, stopping rule, run parameters, mesh tagging and the
history CSV format -- against the reference's golden values and bytes."""

import numpy as np
import pytest

from paper_2601_05709_b200 import ConfigError, IterationRecord, RunParams, adaptive_time, stopping_check
from paper_2601_05709_b200.mesh import build_box_mesh, build_rect_mesh, mesh_diameter
from paper_2601_05709_b200.output import history_header, history_row, write_history_csv
from paper_2601_05709_b200.ppl import lagrangian_value, ppl_init, ppl_update


def test_ppl_table(golden):
    st = ppl_init(1)
    for c, row in zip(golden["ppl_inputs"], golden["ppl_table"]):
        st = ppl_update(st, [c])
        got = [st.z[0], st.lam[0], st.mu[0], st.delta, lagrangian_value(2.0, [c], st)]
        np.testing.assert_allclose(got, row, rtol=1e-15, atol=0)


def test_adaptive_time_hand_example_and_rng(golden):
    quiet = RunParams(random_pars=(1, 0.0))
    t, s = adaptive_time(0.2, quiet, None)  # reference test_driver.py:110-114
    assert t == pytest.approx(0.05, rel=1e-12) and s == 15
    assert adaptive_time(0.0, quiet, None) == (1e-1, 16)
    assert adaptive_time(1e12, quiet, None) == (1e-3, 8)
    rng = np.random.default_rng(1)
    got = [adaptive_time(b, RunParams(), rng) for b in golden["adaptive_btt"]]
    np.testing.assert_array_equal(np.array(got, dtype=float), golden["adaptive_out"])


@pytest.mark.parametrize("kw", [
    {"lv_time": (0.1, 0.1)}, {"lv_time": (0.0, 0.1)}, {"lv_iter": (16, 8)},
    {"random_pars": (1, 1.0)}, {"random_pars": (1, -0.1)}, {"prev": 0}, {"niter": -1},
    {"dfactor": 0.0}, {"reinit_step": 0}, {"reinit_pars": (0, 0.1)}, {"reinit_pars": (8, 0.0)},
    {"cost_tol": 0.0}, {"level_set_scheme": "cn"},
])
def test_run_params_rejects(kw):
    with pytest.raises(ConfigError):
        RunParams(**kw)


def _records(costs, lagr=None, ctrn=None):
    return [IterationRecord(iteration=i, cost=float(c), constraint=np.zeros(0),
                            lagrangian=float(lagr[i]) if lagr is not None else float(c),
                            ctrn_err=float(ctrn[i]) if ctrn is not None else 0.0,
                            multipliers=np.zeros(0)) for i, c in enumerate(costs)]


def test_stopping_rule():
    p = RunParams(start_to_check=2, prev=3, cost_tol=1e-2)
    flat = _records([1.0, 1.0, 1.0, 1.0, 1.0])
    assert not stopping_check(flat[:3], p, False)  # iteration 2 <= start_to_check
    assert stopping_check(flat, p, False)
    assert not stopping_check(_records([1.0, 2.0, 1.0, 1.0]), p, False)
    # constrained: needs ctrn_err < ctrn_tol as well
    assert not stopping_check(_records([1.0] * 5, ctrn=[0.5] * 5), p, True)
    assert stopping_check(_records([1.0] * 5, ctrn=[0.0] * 5), p, True)


def test_history_csv_bytes_match_reference(golden, tmp_path):
    ref = str(golden["run_history_csv"])
    lines = ref.strip("\n").split("\n")
    assert lines[0] == history_header(1)
    recs = []
    for row in lines[1:]:
        c = row.split(",")
        recs.append(IterationRecord(iteration=int(c[0]), cost=float(c[1]), constraint=np.zeros(1),
                                    lagrangian=float(c[2]), ctrn_err=float(c[3]),
                                    multipliers=np.array([float(c[8])]), t_end=float(c[4]),
                                    steps=int(c[5]), form_value=float(c[6]), wall_ms=float(c[7])))
    assert "\n".join(history_row(r) for r in recs) == "\n".join(lines[1:])
    out = tmp_path / "h.csv"
    write_history_csv(out, recs)
    assert out.read_text() == ref


def test_rect_mesh_host_arrays(golden):
    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    m = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 7, 5, rules)
    np.testing.assert_array_equal(m.boundary_facets, golden["mesh_facets"])
    np.testing.assert_array_equal(m.facet_tags, golden["mesh_tags"])
    assert mesh_diameter(m) == golden["mesh_diameter_7x5"][0]
    with pytest.raises(ConfigError):
        build_rect_mesh((0.0, 0.0, 1.0, 1.0), 0, 3)
    with pytest.raises(ConfigError):
        build_rect_mesh((0.0, 0.0, -1.0, 1.0), 3, 3)


def test_box_mesh_facets_match_oracle():
    from oracle.grid import Grid
    m = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), (4, 3, 2), [(1, lambda p: p[:, 0] < 1e-12)])
    g = Grid((0.0, 0.0, 0.0), (2.0, 1.0, 1.0), (4, 3, 2), [(1, lambda p: p[:, 0] < 1e-12)])
    np.testing.assert_array_equal(m.boundary_facets, g.boundary_facets)
    np.testing.assert_array_equal(m.facet_tags, g.facet_tags)
    np.testing.assert_allclose(m.facet_measures, g.facet_measures(), rtol=1e-14)
