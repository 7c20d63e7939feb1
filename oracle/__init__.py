"""CPU oracle for the colour-scheduled sweep — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_1810_04033_b200`) imports this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may use it, and only as the checker
or the timed CPU baseline — never as the thing measured or shipped.

Two independent restatements of the reference algorithm live here:

* `restate.py`  — NumPy strided-slice restatement (Form R bit-exact vs the
  reference `stencil_lab`, Form D / Q1 / patches defined here);
* `sweep_oracle.c` — the same arithmetic as plain C loops (pthreads over the
  rows of one colour), built into `oracle/_build/liboracle.so`;
  it is the fast checker at large sizes and the CPU baseline ("port").

Parity pin: Form R is pinned bit-for-bit against the reference itself
(`tests/golden/make_golden.py` imports `/root/reference/pkg/src` in the build
container and commits digests).  Form D, FE27-Q1 and batched patches have no
reference counterpart: they are pinned only by agreement of
the two restatements here — "parity self-pinned".
"""
