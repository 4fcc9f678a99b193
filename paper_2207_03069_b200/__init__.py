"""B200-native DABS hot path (arXiv 2207.03069): C ABI (include/dabs.h) over
hand-written sm_100a CUDA kernels, with a thin ctypes binding.

    from paper_2207_03069_b200 import Solver
    E, x = Solver(W, s_milli=100, b_milli=10000).run(seed=1, flip_budget=10**9)
"""
from .dabs import DabsError, Solver, load, torch_exchange  # noqa: F401

ALGORITHMS = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor"]
GENOPS = ["Mutation", "Crossover", "Xrossover", "Zero", "One", "IntervalZero", "Best", "Random"]
