"""Final-map quality parity (SPEC acceptance / north-star correctness part 3):
the GPU fit (throughput SGD, GPU PCA, bf16 or exact kNN) reaches the
reference's NP@10 and random-triplet accuracy on identical data, measured by
the reference's own metric code (metrics.hpp:113-243, via oracle/_ref)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("knn_mode", ["exact", "bf16"])
def test_quality_matches_reference(port, ref, ctx, knn_mode):
    import paper_2505_15511_b200 as nb
    from oracle import train_config
    x = port.gaussian_mixture(6000, 32, 10, 10.0, 42)
    kw = dict(epochs=100, workers=2, n_clusters=6)
    r7 = ref.fit(x, train_config(seed=7, **kw))["layout"]
    r8 = ref.fit(x, train_config(seed=8, **kw))["layout"]
    g7 = nb.fit(x, nb.TrainConfig(seed=7, sgd_mode="hogwild", knn_mode=knn_mode, **kw), ctx=ctx)
    np_r7, _ = ref.neighborhood_preservation(x, r7, 10)
    np_r8, _ = ref.neighborhood_preservation(x, r8, 10)
    np_g, _ = ref.neighborhood_preservation(x, g7, 10)
    t_r7, se = ref.random_triplet_accuracy(x, r7, 100000, 1)
    t_r8, _ = ref.random_triplet_accuracy(x, r8, 100000, 1)
    t_g, _ = ref.random_triplet_accuracy(x, g7, 100000, 1)
    print(f"NP@10 ref {np_r7:.4f}/{np_r8:.4f} gpu {np_g:.4f}; triplet ref {t_r7:.4f}/{t_r8:.4f} "
          f"gpu {t_g:.4f}")
    assert abs(np_g - np_r7) <= max(0.02, 3 * abs(np_r7 - np_r8))
    assert abs(t_g - t_r7) <= max(0.02, 3 * abs(t_r7 - t_r8), 5 * se)
