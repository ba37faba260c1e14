"""paper_1801_09661_b200 — B200-native hot path of OEM penalized regression on tall data
(arXiv 1801.09661): Gram / fold-Gram / weighted-Gram passes on the FP64 tensor cores, the sparse
(CSR) Gram pass, the certified d rule, and persistent OEM path solvers, behind the C ABI in
include/oem.h."""
from .oem import (Context, CvResult, LogisticResult, OemError, PathResult, oem_fit_logistic, oem_fit_path,  # noqa: F401
                  oem_cv_error, oem_gram, oem_gram_csr, oem_gram_folds, oem_gram_folds_host, oem_gram_folds_sums, oem_gram_host, oem_gram_moments, oem_gram_sums, oem_logit_grad, oem_path_loss,
                  oem_gram_weighted, oem_nccl_unique_id)
