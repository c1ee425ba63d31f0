"""Plain containers for the three inputs of the hot path.

The paper's problem statement: the system "takes a cluster resource
specification, a set of models, and a periodic workload profile" and
searches for a placement = "a specific cluster group partition, model
selection, and parallel configuration".

Units: times are int64 nanoseconds, sizes int64 bytes (reading C19).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Problem:
    """Models x parallel configs, plus the cluster.

    stage_ns[m, p, k]  occupancy of pipeline stage k of model m under config p
                       (k < cfg_stages[p]; entries beyond are 0)
    tail_ns[m, p]      overhead added to the finish time only (reading C4)
    mem_bytes[m, p]    bytes per device of one replica; < 0 = not placeable
    slo_ns[m]          per-request deadline offset ("SLO scale")
    """

    model_names: list
    configs: list  # [(s, n)] inter-op stages s, intra-op degree n
    slo_ns: np.ndarray  # int64 [M]
    stage_ns: np.ndarray  # int64 [M, P, S]
    tail_ns: np.ndarray  # int64 [M, P]
    mem_bytes: np.ndarray  # int64 [M, P]
    num_devices: int
    budget_bytes: int
    meta: dict = field(default_factory=dict)

    @property
    def num_models(self) -> int:
        return len(self.model_names)

    @property
    def num_configs(self) -> int:
        return len(self.configs)

    @property
    def max_stages(self) -> int:
        return int(self.stage_ns.shape[2])

    @property
    def cfg_stages(self) -> np.ndarray:
        return np.array([s for s, _ in self.configs], dtype=np.int32)

    @property
    def cfg_devices(self) -> np.ndarray:
        return np.array([s * n for s, n in self.configs], dtype=np.int32)

    def with_slo_scale(self, scale: float) -> "Problem":
        """Same problem with slo_ns = round(scale * D_m) (reading C10)."""
        base = np.asarray(self.meta["latency_ns"], dtype=np.float64)
        slo = np.rint(base * float(scale)).astype(np.int64)
        return Problem(self.model_names, self.configs, slo, self.stage_ns,
                       self.tail_ns, self.mem_bytes, self.num_devices,
                       self.budget_bytes, dict(self.meta, slo_scale=scale))

    def validate(self) -> None:
        M, P, S = self.stage_ns.shape
        assert len(self.model_names) == M and len(self.configs) == P
        assert self.slo_ns.shape == (M,) and self.slo_ns.dtype == np.int64
        assert self.tail_ns.shape == (M, P) and self.mem_bytes.shape == (M, P)
        for p, (s, n) in enumerate(self.configs):
            assert 1 <= s <= S and n >= 1
            assert np.all(self.stage_ns[:, p, s:] == 0)
        assert np.all(self.stage_ns >= 0) and np.all(self.tail_ns >= 0)
        assert np.all(self.slo_ns >= 0)


@dataclass
class Trace:
    """Time-sorted workload W: arrival_ns non-decreasing, model ids."""

    arrival_ns: np.ndarray  # int64 [N]
    model: np.ndarray  # int32 [N]
    meta: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return int(self.arrival_ns.shape[0])

    def prefix(self, n: int) -> "Trace":
        return Trace(self.arrival_ns[:n].copy(), self.model[:n].copy(), dict(self.meta, prefix=n))

    def until(self, t_ns: int) -> "Trace":
        n = int(np.searchsorted(self.arrival_ns, t_ns, side="left"))
        return self.prefix(n)


@dataclass
class Placement:
    """One candidate placement: groups with a config each, and the model
    selection per group.  group_cfg[g] = config id, or -1 = no group.
    host_mask[m] bit g set <=> group g hosts a replica of model m."""

    group_cfg: np.ndarray  # int32 [G]
    host_mask: np.ndarray  # uint64 [M]

    @property
    def num_groups(self) -> int:
        return int(self.group_cfg.shape[0])

    def hosts(self, m: int) -> list:
        mask = int(self.host_mask[m])
        return [g for g in range(self.num_groups) if (mask >> g) & 1]

    def models_on(self, g: int) -> list:
        return [m for m in range(self.host_mask.shape[0]) if (int(self.host_mask[m]) >> g) & 1]

    @staticmethod
    def from_lists(group_cfg, groups_models, num_models) -> "Placement":
        """groups_models[g] = iterable of model ids hosted on group g."""
        mask = np.zeros(num_models, dtype=np.uint64)
        for g, ms in enumerate(groups_models):
            for m in ms:
                mask[m] |= np.uint64(1) << np.uint64(g)
        return Placement(np.asarray(group_cfg, dtype=np.int32), mask)
