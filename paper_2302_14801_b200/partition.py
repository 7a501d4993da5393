"""Drop-in for `lodforge.partition` (reference partition.py:79-302) on the B200.

`partition(cloud, config)` and `Partitioner(cloud, config, bounds).run()` keep the
reference's signatures, defaults and exceptions; the hierarchical counting sort runs
in `liblodb200.so` (count -> extension rounds -> merge pyramid -> node table ->
stable distribute).  The result is a `GpuOctree`.
"""
from __future__ import annotations

from .device import DeviceTree, make_config
from .model import AABB, BuildConfig, Octree, PointCloud
from .octree import GpuOctree

UNMERGEABLE = 0xFFFFFFFF  # reference partition.py:20


class Partitioner:
    """Mirror of the reference Partitioner's composite entry (`run`, partition.py:291-297).

    The stage-level methods of the reference (count/merge/...) are fused on the device;
    only the composite is exposed.  `bounds` forces the world cube (partition.py:82,87).
    """

    def __init__(self, cloud: PointCloud, config: BuildConfig, bounds: AABB | None = None,
                 device_tree: DeviceTree | None = None):
        if len(cloud) == 0:
            raise ValueError("cannot partition an empty point cloud")
        self.cloud = cloud
        self.config = config
        self.bounds = bounds
        self._dev = device_tree

    def run(self) -> Octree:
        dev = self._dev or DeviceTree()
        cfg = self.config
        d_rec, fmt, n = dev.upload(self.cloud.positions, self.cloud.colors)
        b = None if self.bounds is None else (*self.bounds.min, self.bounds.size)
        dev.split(d_rec, n, fmt, make_config(cfg.T, cfg.initial_depth, cfg.extension_depth, cfg.max_depth), b)
        return GpuOctree(dev, cfg)


def partition(cloud: PointCloud, config: BuildConfig | None = None) -> Octree:
    """Partition a point cloud into an octree with at most T points per leaf (partition.py:300-302)."""
    return Partitioner(cloud, config or BuildConfig()).run()
