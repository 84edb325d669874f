"""Body of __graft_entry__.smoke() (filled in as the engine lands)."""


def run_smoke():
    import numpy as np

    import paper_2508_04462_b200 as card
    from oracle import card_oracle as O

    cache = card.TreeCache(0, card.CacheConfig(K=4, k=2, max_depth=3))
    twin = O.SoATree(0, 4, 2, 3, log_fn=O.cr_log)
    d = np.array([[0.5, 0.3, 0.2]])
    cache.expand_layer(d)
    twin.expand(d)
    assert cache.frontier == twin.frontier
