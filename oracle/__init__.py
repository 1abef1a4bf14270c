"""CPU oracle for the MaxSim / Col-Bandit hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference's algorithm (arxiv 2602.02827, package
``colbandit`` 0.1.0 under /root/reference/pkg/src/colbandit) on the CPU so
the CUDA path can be checked against it. It is the checker, never the thing
measured or shipped: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_2602_02827_b200`` never imports it and has no CPU
fallback.

Pinning: every function here is checked against golden vectors produced by
running the unmodified reference in the build container
(``tests/golden/make_golden.py``; fixtures in ``tests/golden/``), see
``tests/test_oracle_golden.py``. The RNG stream (numpy ``Generator(PCG64)``,
numpy 2.3.5, a third-party dependency of the reference) is pinned by golden
streams drawn from numpy itself.

Modules:
    maxsim_ref  — exhaustive scorer: cells, exactly-rounded scores, Top-K.
    bandit_ref  — the Col-Bandit adaptive loop (``run``) and ``full_rerank``.
    pcg64_ref   — PCG64 XSL-RR 128/64 + numpy's random()/integers(n) draws.
"""
