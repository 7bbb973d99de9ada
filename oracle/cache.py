"""The temporal window ("window ... the earliest value is
evicted"): a bounded FIFO of frozen
parameter snapshots keyed by strictly increasing timesteps."""
import collections

import numpy as np


class Window:
    def __init__(self, capacity):
        if capacity <= 0:
            raise ValueError("capacity must be >= 1")
        self.capacity = int(capacity)
        self.items = collections.deque()

    def insert(self, timestep, params_list):
        """Copy the snapshot in; returns the evicted timestep or -1."""
        if self.items and timestep <= self.items[-1][0]:
            raise ValueError("timesteps must be strictly increasing")
        evicted = -1
        if len(self.items) == self.capacity:
            evicted = self.items.popleft()[0]
        self.items.append((int(timestep), [np.array(p, copy=True) for p in params_list]))
        return evicted

    def evict(self):
        if not self.items:
            raise LookupError("evict on an empty window")
        return self.items.popleft()[0]

    def timesteps(self):
        return [t for t, _ in self.items]
