"""Map quality of a throughput-SGD build variant (NOMAD_B200_LIB=<variant>.so):
NP@10 / random-triplet accuracy by the reference's metric code (oracle/_ref).
python tools/hog_quality.py [n] [d] [blobs] [epochs]"""
import json
import sys

sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402
from oracle import Oracle  # noqa: E402


def main():
    n, d, blobs, epochs = (int(a) for a in (sys.argv[1:] + ["20000", "32", "10", "200"][len(sys.argv) - 1:]))
    port, ref = Oracle("port"), Oracle("reference")
    x = port.gaussian_mixture(n, d, blobs, 10.0, 42)
    ctx = nb.Context(0)
    out = {"n": n, "d": d, "blobs": blobs, "epochs": epochs}
    for seed in (7, 8):
        y = nb.fit(x, nb.TrainConfig(seed=seed, epochs=epochs, workers=8, n_clusters=8,
                                     sgd_mode="hogwild", knn_mode="bf16"), ctx=ctx)
        npk, _ = ref.neighborhood_preservation(x, y, 10, sample=min(n, 4000), seed=1)
        out[f"np10_s{seed}"] = round(float(npk), 4)
        out[f"triplet_s{seed}"] = round(ref.random_triplet_accuracy(x, y, 20000, 3)[0], 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
