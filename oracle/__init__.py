"""CPU oracle for the H_eff·ψ / renormalization path — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference algorithm (sector_dmrg, the
arxiv 2305.05581 artifact under /root/reference/pkg/src/sector_dmrg), each
function citing the reference file:line it follows.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the
timed CPU baseline — never as part of the product path, which has no CPU
fallback.

Pinning: ``tests/golden/*.npz`` hold outputs of the reference itself
(imported from /root/reference in the build container by
``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks this
restatement against them (grouping bit-exact, σ/energies to 1e-12).
"""
