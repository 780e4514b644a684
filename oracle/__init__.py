"""CPU fp64 oracle for the 3D-PMM FC layer of AxoNN (arXiv 2502.08145).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute anything under ``oracle/``.  The only permitted callers are
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py``.  The oracle shares no code with the
CUDA path (``paper_2502_08145_b200``); both read seeded inputs from
``synthdata`` only.

Modules (each function cites the PAPER.md passage it follows):

* ``fc``         — the unsharded layer: O = I·W, dI = dO·Wᵀ, dW = Iᵀ·dO
                   (§IV-A "3D PMM").
* ``grid``       — the 4D virtual grid, rank <-> (i,j,k,d), process groups and
                   configuration enumeration.
* ``ring``       — ring all-gather / reduce-scatter / all-reduce, step by step,
                   with per-rank byte accounting (PAPER.md:443-445,
                   Assumption-1; Thakur et al. ring algorithm).
* ``alg1``       — Algorithm 1 simulated over every rank of a grid
                   (PAPER.md:368-393), transposed layers,
                   and the data-parallel gradient all-reduce.
* ``perf_model`` — Eqs. 1-7 and the ranked configuration list
                   (PAPER.md:458-597).
* ``flops``      — model-flop accounting and % of peak.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; see DESIGN.md "Oracle pins".  The only parity
unpinned quantities are hardware measurements (Case-1 bandwidth table values)
which the oracle takes as inputs and never computes.
"""
