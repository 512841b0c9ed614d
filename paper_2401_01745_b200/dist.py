"""Multi-process (one process per GPU) z-slab runs. Implemented in a later
step; see DESIGN.md §6."""


def bench_main(*a, **k):
    raise NotImplementedError("multi-GPU z-slab bench is not implemented yet")
