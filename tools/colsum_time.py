"""Sequential-sum kernels (k_seq_colsum2: LSH data mean and k-means centroid sums; k_pca_cols:
exact PCA applies) on 2M x 768: run under ncu to time them."""
import sys
sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402
ctx = nb.Context(0)
x = nb.generate_mixture(2000000, 768, 16, 10.0, 42, ctx=ctx)
c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 16, 7, ctx=ctx), 100, ctx=ctx)
x2 = nb.generate_mixture(50000, 768, 16, 10.0, 42, ctx=ctx)
nb.pca_init(x2, 7, ctx=ctx)
