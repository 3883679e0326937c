"""The knob grid of one sweep: L power budgets over one set of knob values.

The reference re-enumerates the legal configs of ONE budget inside every
``optimize_corun`` call (hwopt.py:57, core.py:380-397) and every solo split
inside every ``solorun_time`` call (estimator.py:164).  Here the enumeration is
done once per sweep, on the host, for up to ``MAX_BUDGETS`` budgets at once:

* the co-run configs of all budgets are merged into one *union* list kept in
  the reference's lexicographic order, so each budget's own list is an
  order-preserving subsequence and first-index tie-breaking carries over;
* ``mask[c]`` has bit ``l`` set when config ``c`` is legal in budget ``l``
  (the total-power mask, core.py:388,394);
* ``knob1``/``knob2`` are the 4 normalized knob inputs (core.py:368-371) of the
  member-1 view and the reversed-partition member-2 view (core.py:152-159,
  estimator.py:122);
* solo splits (core.py:400-407) are stacked per budget with offsets.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .core import ConfigSpace, ValidationError, corun_tuples, enumerate_solo_splits, knob_vector

MAX_BUDGETS = 8


class KnobGrid:
    def __init__(self, spaces: Sequence[ConfigSpace]):
        spaces = tuple(spaces)
        if not 1 <= len(spaces) <= MAX_BUDGETS:
            raise ValidationError(f"a sweep covers 1..{MAX_BUDGETS} budgets, got {len(spaces)}")
        ref = spaces[0]
        for sp in spaces[1:]:
            if (sp.cpu_partitions, sp.gpu_partitions, sp.cpu_caps, sp.gpu_caps) != \
               (ref.cpu_partitions, ref.gpu_partitions, ref.cpu_caps, ref.gpu_caps):
                raise ValidationError("budgets swept together must share the knob value sets")
        self.spaces = spaces
        per_budget = [set(corun_tuples(sp)) for sp in spaces]
        # union in cartesian (reference) order
        union = [t for t in corun_tuples(ConfigSpace(
            cpu_partitions=ref.cpu_partitions, gpu_partitions=ref.gpu_partitions,
            cpu_caps=ref.cpu_caps, gpu_caps=ref.gpu_caps, p_total=ref.p_max, p_max=ref.p_max,
            cap_sum_levels=tuple(sorted({lv for sp in spaces for lv in sp.active_levels}))))
            if any(t in s for s in per_budget)]
        self.configs = union
        G = len(union)
        self.mask = np.zeros(G, dtype=np.uint32)
        self.local_index = np.full((len(spaces), G), -1, dtype=np.int32)
        self.budget_configs = []          # per budget: grid indices in its own order
        for l, s in enumerate(per_budget):
            idx = [g for g, t in enumerate(union) if t in s]
            self.mask[idx] |= np.uint32(1 << l)
            self.local_index[l, idx] = np.arange(len(idx), dtype=np.int32)
            self.budget_configs.append(np.asarray(idx, dtype=np.int32))
        self.n_configs = [len(ix) for ix in self.budget_configs]
        self.knob1 = np.array([knob_vector(cp, gp, cc, gc) for cp, gp, cc, gc in union],
                              dtype=np.float64).reshape(G, 4)
        self.knob2 = np.array([knob_vector(cp[::-1], gp[::-1], cc, gc) for cp, gp, cc, gc in union],
                              dtype=np.float64).reshape(G, 4)
        self.solo_splits = [enumerate_solo_splits(sp) for sp in spaces]
        offs = [0]
        for sp_list in self.solo_splits:
            offs.append(offs[-1] + len(sp_list))
        self.solo_offsets = offs
        rows = [(1.0, 1.0, c / 250.0, g / 250.0) for sl in self.solo_splits for c, g in sl]
        # solo view: partitions (32,0)/(8,0) -> 32/32 = 8/8 = 1 (core.py:179-181, 368-371)
        self.solo_knob = np.array(rows, dtype=np.float64).reshape(len(rows), 4)

    @property
    def n_grid(self) -> int:
        return len(self.configs)

    @property
    def n_budgets(self) -> int:
        return len(self.spaces)

    def check_nonempty(self, corun: bool = True, solo: bool = True) -> None:
        """The reference's errors for an empty search (hwopt.py:62-64, estimator.py:165-167)."""
        for l, sp in enumerate(self.spaces):
            if corun and self.n_configs[l] == 0:
                raise ValidationError(f"no co-run configs exist for p_total {sp.p_total}")
            if solo and self.solo_offsets[l + 1] == self.solo_offsets[l]:
                raise ValidationError(f"p_total {sp.p_total} is unreachable on the cap grids")

    def units_per_pair(self) -> int:
        """Reference-equivalent (pair, config) evaluations per pair: sum over budgets."""
        return int(sum(self.n_configs))
