#!/usr/bin/env python
"""Run the tree-prior kernel a few times at C2 size (for ncu)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    torch.cuda.set_device(0)
    n, d = 5392, 2
    parent, t = workload.coalescent_forest(n, 1, 0.0, seed=11)
    w = workload.config("C2")
    with mds.MDS(n, d, stream=torch.cuda.current_stream()) as c:
        c.set_locations(w.x0)
        c.set_tree_prior(parent, t)
        for _ in range(3):
            c.tree_prior()
    print("ok")


if __name__ == "__main__":
    main()
