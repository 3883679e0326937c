"""Host logic of the boundary: enumeration, knob grid, normalization, fnn I/O. CPU.

The known-answer checks restate the reference's own tests
(pkg/tests/test_core.py:165-290, test_fnn.py) against this package.
"""

import json

import numpy as np
import pytest

from paper_2405_03831_b200 import core, fnn
from paper_2405_03831_b200.core import ConfigSpace, HardwareConfig, ValidationError
from paper_2405_03831_b200.grid import KnobGrid


def test_corun_counts_match_implementation_not_spec():
    assert len(core.enumerate_corun_configs(core.default_space(400.0))) == 100
    assert len(core.enumerate_corun_configs(core.default_space(350.0))) == 50  # SPEC says 60
    assert core.enumerate_corun_configs(core.default_space(240.0)) == []


def test_independent_recount():
    for p in (250.0, 300.0, 350.0, 375.0, 400.0, 450.0):
        sp = core.default_space(p)
        levels = {lv for lv in sp.cap_sum_levels if lv <= p}
        caps = sum(1 for c in core.CPU_CAPS for g in core.GPU_CAPS if c + g in levels)
        assert len(core.enumerate_corun_configs(sp)) == 5 * 2 * caps


def test_lexicographic_order():
    cfgs = core.enumerate_corun_configs(core.default_space(400.0))
    keys = [(core.CPU_PARTITIONS.index(h.cpu_partition), core.GPU_PARTITIONS.index(h.gpu_partition),
             core.CPU_CAPS.index(h.cpu_cap), core.GPU_CAPS.index(h.gpu_cap)) for h in cfgs]
    assert keys == sorted(keys)
    assert all(h.is_corun and h.cap_sum <= 400 for h in cfgs)


def test_solo_splits_exact():
    assert core.enumerate_solo_splits(core.default_space(350.0)) == [
        (100.0, 250.0), (125.0, 225.0), (150.0, 200.0), (175.0, 175.0), (200.0, 150.0)]
    assert core.enumerate_solo_splits(core.default_space(400.0)) == [
        (150.0, 250.0), (175.0, 225.0), (200.0, 200.0), (225.0, 175.0), (250.0, 150.0)]


def test_reversed_partitions_and_validation():
    hc = HardwareConfig((3 * 8, 8), (3, 4), 150, 250)
    r = hc.reversed_partitions()
    assert r.cpu_partition == (8, 24) and r.gpu_partition == (4, 3) and r.cpu_cap == 150.0
    with pytest.raises(ValidationError, match="cpu_partition"):
        HardwareConfig((1, 31), (3, 4), 150, 250)
    with pytest.raises(ValidationError, match="gpu_cap"):
        HardwareConfig((2, 30), (3, 4), 150, 260)


def test_normalize_input_known_answers():
    b = np.full(36, 10.0)
    j1 = core.JobProfile("a", np.full(18, 5.0), 20.0)
    j2 = core.JobProfile("b", np.full(18, 50.0), 20.0)
    solo = core.normalize_input(j1, None, core.solo_config(250, 250), core.default_space(), b)
    assert np.array_equal(solo[:4], [1, 1, 1, 1]) and np.all(solo[22:] == 0) and np.all(solo[4:22] == 0.5)
    x = core.normalize_input(j1, j2, HardwareConfig((16, 16), (4, 3), 125, 200), core.default_space(), b)
    assert x[0] == 0.5 and x[1] == 0.5 and x[2] == 0.5 and x[3] == 0.8 and np.all(x[22:] == 1.0)
    with pytest.raises(ValidationError, match="bounds entry 3"):
        bb = b.copy(); bb[3] = 0
        core.normalize_input(j1, None, core.solo_config(250, 250), core.default_space(), bb)


def test_knob_grid_single_budget_matches_enumeration():
    sp = core.default_space(400.0)
    g = KnobGrid([sp])
    assert [HardwareConfig(*t) for t in g.configs] == core.enumerate_corun_configs(sp)
    assert np.all(g.mask == 1) and g.n_configs == [100]
    hc = core.enumerate_corun_configs(sp)[7]
    assert np.array_equal(g.knob1[7], [hc.cpu_partition[0] / 32, hc.gpu_partition[0] / 8,
                                       hc.cpu_cap / 250, hc.gpu_cap / 250])
    r = hc.reversed_partitions()
    assert np.array_equal(g.knob2[7], [r.cpu_partition[0] / 32, r.gpu_partition[0] / 8,
                                       r.cpu_cap / 250, r.gpu_cap / 250])
    assert np.array_equal(g.solo_knob[:, :2], np.ones((5, 2)))


def test_knob_grid_union_preserves_each_budget_order():
    levels = (300, 325, 350, 375, 400)
    spaces = [ConfigSpace(p_total=p, cap_sum_levels=levels) for p in (300.0, 325.0, 350.0, 375.0, 400.0)]
    g = KnobGrid(spaces)
    assert g.n_grid == 220 and g.n_configs == [30, 70, 120, 170, 220]
    assert [g.solo_offsets[k + 1] - g.solo_offsets[k] for k in range(5)] == [3, 4, 5, 5, 5]
    for l, sp in enumerate(spaces):
        own = core.enumerate_corun_configs(sp)
        assert [HardwareConfig(*g.configs[k]) for k in g.budget_configs[l]] == own
        assert np.array_equal(g.local_index[l][g.budget_configs[l]], np.arange(len(own)))
    with pytest.raises(ValidationError, match="share"):
        KnobGrid([core.default_space(), ConfigSpace(cpu_caps=(100, 150))])


def test_fine_grid_needs_no_patch_for_the_sweep_but_configs_do():
    fine_c = tuple(100.0 + 6.25 * k for k in range(25))
    fine_g = tuple(150.0 + 6.25 * k for k in range(17))
    g = KnobGrid([ConfigSpace(cpu_caps=fine_c, gpu_caps=fine_g, p_total=400.0)])
    assert g.n_grid == 340 and len(g.solo_splits[0]) == 17
    with pytest.raises(ValidationError):
        HardwareConfig(*g.configs[1])       # caps validated against module constants


def test_weights_roundtrip_and_errors(tmp_path, weights):
    p = tmp_path / "w.json"
    fnn.save_weights(weights, p)
    w2 = fnn.load_weights(p)
    for k in ("w1", "b1", "w2", "b2", "w_out", "b_out", "feature_bounds"):
        assert np.array_equal(getattr(w2, k), getattr(weights, k))
    doc = json.loads(p.read_text())
    doc["version"] = 2
    p.write_text(json.dumps(doc))
    with pytest.raises(ValidationError, match="version"):
        fnn.load_weights(p)
    doc["version"] = 1
    del doc["layer_2"]
    p.write_text(json.dumps(doc))
    with pytest.raises(ValidationError, match="missing field"):
        fnn.load_weights(p)
    p.write_text("{not json")
    with pytest.raises(ValidationError, match="not valid JSON"):
        fnn.load_weights(p)


def test_initialize_weights_is_seeded():
    a = fnn.initialize_weights(3, np.ones(36))
    b = fnn.initialize_weights(3, np.ones(36))
    assert np.array_equal(a.w1, b.w1) and a.b_out[0] == 1.0 and np.all(a.b1 == 0)


def test_schedule_and_jobset_validation():
    with pytest.raises(ValidationError):
        core.SchedulingParams(window=3)
    with pytest.raises(ValidationError):
        core.JobSet(())
    j = core.JobProfile("x", np.ones(18), 10.0)
    with pytest.raises(ValidationError, match="not finite"):
        core.JobProfile("y", np.r_[np.ones(17), np.nan], 10.0)
    with pytest.raises(ValidationError, match="base_time"):
        core.JobProfile("y", np.ones(18), 0.0)
    s = core.Schedule((core.JobSet((j,)),), ((core.solo_config(200, 200),),), (False,))
    s.validate_against([j], core.default_space())
