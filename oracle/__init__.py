"""oracle/ — CPU restatement of the reference's hot-path algorithms.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / --impl reference legs may import this package, and only as the
checker or the timed reference arm — never as the thing measured or shipped.
The product (paper_2411_09982_b200) never imports it and has no CPU fallback.

The reference (/root/reference/pkg/src/effham) is pure numpy/scipy; these
modules restate its arithmetic statement by statement so results are
bit-identical on the same host (each function cites the file:line it
follows).  Parity pinning: tests/test_oracle_golden.py checks this
restatement bit-for-bit against golden vectors produced by running the
reference itself (oracle/gen_golden.py -> tests/golden/*.npz).

The second-order Magnus term has NO reference implementation:
``magnus_oracle.second_order_coefficients`` is the builder's restatement of
SURVEY.md Appendix B — parity for it is UNPINNED by the reference and is
instead checked against brute-force nested quadrature
(tests/test_second_order_oracle.py).
"""
