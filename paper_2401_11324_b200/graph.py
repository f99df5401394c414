"""Graph container with the reference's layout and checks (graph.py:20-104).

Adjacency is a padded (node_count, degree_bound) int32 matrix with
``NO_NODE = -1`` padding plus one degree per node and a medoid entry point.
The offline Vamana builder is out of scope; the GPU tooling
in ``tools/`` builds graphs for the benchmarks.
"""

from __future__ import annotations

import numpy as np

from .errors import ParameterError

NO_NODE = -1


class GraphIndex:
    def __init__(self, adjacency, degrees, medoid: int, degree_bound: int | None = None,
                 validate: bool = True):
        adjacency = np.ascontiguousarray(adjacency, dtype=np.int32)
        degrees = np.ascontiguousarray(degrees, dtype=np.int32)
        if adjacency.ndim != 2 or degrees.shape != (adjacency.shape[0],):
            raise ParameterError("adjacency must be (n, R) with one degree per node")
        self.adjacency = adjacency
        self.degrees = degrees
        self.medoid = int(medoid)
        self.degree_bound = int(degree_bound if degree_bound is not None else adjacency.shape[1])
        if validate:
            self.validate()

    @property
    def node_count(self) -> int:
        return self.adjacency.shape[0]

    @classmethod
    def from_lists(cls, neighbour_lists, medoid: int, degree_bound: int) -> "GraphIndex":
        n = len(neighbour_lists)
        adjacency = np.full((n, degree_bound), NO_NODE, dtype=np.int32)
        degrees = np.zeros(n, dtype=np.int32)
        for i, ids in enumerate(neighbour_lists):
            ids = np.asarray(ids, dtype=np.int32)
            if ids.size > degree_bound:
                raise ParameterError(f"node {i} has {ids.size} neighbours, bound is {degree_bound}")
            adjacency[i, :ids.size] = ids
            degrees[i] = ids.size
        return cls(adjacency, degrees, medoid, degree_bound)

    def neighbours(self, node: int) -> np.ndarray:
        return self.adjacency[node, :self.degrees[node]]

    def neighbour_lists(self):
        return [self.adjacency[i, :self.degrees[i]].copy() for i in range(self.node_count)]

    def validate(self) -> None:
        """graph.py:69-90: range, degree, self-loop and duplicate checks."""
        n = self.node_count
        if n == 0:
            raise ParameterError("graph must contain at least one node")
        if not (0 <= self.medoid < n):
            raise ParameterError(f"medoid {self.medoid} out of range for {n} nodes")
        if np.any(self.degrees < 0) or np.any(self.degrees > self.degree_bound):
            raise ParameterError("node degree outside [0, degree_bound]")
        cols = np.arange(self.adjacency.shape[1])
        live = cols[None, :] < self.degrees[:, None]
        ids = self.adjacency[live]
        if ids.size:
            if ids.min() < 0 or ids.max() >= n:
                raise ParameterError("adjacency id out of range")
            rows = np.broadcast_to(np.arange(n)[:, None], self.adjacency.shape)[live]
            if np.any(ids == rows):
                raise ParameterError("self-loop in adjacency")
            srt = np.sort(np.where(live, self.adjacency, np.int32(-1)), axis=1)
            if np.any((srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)):
                raise ParameterError("duplicate neighbour id within a list")

    def __eq__(self, other) -> bool:
        if not isinstance(other, GraphIndex):
            return NotImplemented
        if (self.node_count != other.node_count or self.medoid != other.medoid
                or self.degree_bound != other.degree_bound
                or not np.array_equal(self.degrees, other.degrees)):
            return False
        live = np.arange(self.adjacency.shape[1])[None, :] < self.degrees[:, None]
        return np.array_equal(self.adjacency[live], other.adjacency[:, :self.adjacency.shape[1]][live])


def compute_medoid(vectors) -> int:
    """Id of the point nearest the arithmetic centroid (graph.py:107-115)."""
    x = np.asarray(vectors)
    if x.shape[0] == 0:
        raise ParameterError("cannot compute a medoid of an empty store")
    xf = x.astype(np.float64)
    diff = xf - xf.mean(axis=0)
    return int(np.argmin(np.einsum("nd,nd->n", diff, diff)))
