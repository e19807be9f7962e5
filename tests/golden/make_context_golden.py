"""Record the reference PartitionContext (partitioner.py:95-138) on seeded
random nestings -> tests/golden/context.json.

    PYTHONPATH=/tmp/refpkg/src python tests/golden/make_context_golden.py
"""

import json
import os

import numpy as np

from minispmd.partitioner import PartitionContext

HERE = os.path.dirname(os.path.abspath(__file__))


def _split(rng, ids):
    """Random partition of ``ids`` into equal-size groups."""
    n = len(ids)
    sizes = [s for s in range(1, n + 1) if n % s == 0]
    size = int(rng.choice(sizes))
    perm = [int(i) for i in rng.permutation(ids)]
    return [sorted(perm[i:i + size]) for i in range(0, n, size)]


def main():
    cases = []
    for seed in range(60):
        rng = np.random.default_rng(seed)
        n = int(rng.choice([1, 2, 4, 8, 16]))
        ctx = PartitionContext.root(n)
        steps = []
        for _ in range(int(rng.integers(1, 4))):
            logical = list(range(ctx.num_logical))
            query = _split(rng, logical)
            merge = _split(rng, logical)
            steps.append({"query": query, "physical": ctx.physical_subgroups(query),
                          "merge": merge})
            ctx = ctx.child(merge)
            steps[-1]["groups"] = ctx.device_groups
            steps[-1]["num_logical"] = ctx.num_logical
        cases.append({"n": n, "steps": steps})
    with open(os.path.join(HERE, "context.json"), "w") as f:
        json.dump(cases, f, sort_keys=True)
    print("cases:", len(cases))


if __name__ == "__main__":
    main()
