"""Shared helpers for the GPU parity tests."""

from __future__ import annotations

import numpy as np

from paper_2602_02827_b200 import workloads as W


def case_doc_list(case: W.QueryCase):
    off = case.doc_offsets
    return [case.doc_tokens[off[i]:off[i + 1]] for i in range(case.n_docs)]


def storage_dtype(dt: str):
    return {"f32": None, "f16": None, "bf16": "bf16"}[dt]


def batch_of_cases(cases, clamp_negative=False):
    from paper_2602_02827_b200.batch import TokenBatch

    dt = cases[0].dtype
    return TokenBatch.from_host([c.query for c in cases], [case_doc_list(c) for c in cases],
                                dtype=storage_dtype(dt), clamp_negative=clamp_negative)


def topk_matches(got, ref, ref_scores, rtol):
    """Top-K order equal to the reference except where reference scores tie within ``rtol``."""
    got = list(got)
    ref = list(ref)
    if got == ref:
        return True
    if len(got) != len(ref) or len(set(got)) != len(got):
        return False
    s = np.asarray(ref_scores, dtype=np.float64)
    for g, r in zip(got, ref):
        if g == r:
            continue
        if abs(s[g] - s[r]) > rtol * max(abs(s[r]), 1e-12):
            return False
    return True
