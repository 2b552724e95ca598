"""fp64 CPU oracle for Fast Fourier-Bessel steerable PCA (arXiv 1412.0781).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1412_0781_b200``) never imports it and
shares no code, tables or constants with it.

Everything here is a plain, slow, obviously-correct restatement of the paper
(``P:n`` = line n of PAPER.md), in float64, using numpy/scipy primitives
(``scipy.special.jv``, ``scipy.optimize.brentq``, ``numpy.polynomial.legendre.
leggauss``, ``numpy.fft``, ``numpy.linalg.eigh``, BLAS matmul) as single steps.

Readings of the paper where it is silent, garbled or inconsistent are listed in
DESIGN.md (section "Readings"); the ones that change arithmetic are:

* Q1  Eq. (nufft) is taken with a UNIT prefactor (no 1/(2R)^2).
* Q3  array axis 0 is i1 (multiplies xi_1 = xi cos theta); index i = a - floor(L/2).
* Q8  the k=0 imaginary residue is set to zero.
* Q9  covariance divisor 1/n, centring of k=0 only.
* Q10 eigenvector sign: the entry of largest |u(q)| is made positive (ties -> lowest q).
* Q13 Wiener weight h = l/(l+sigma^2), l = (lambda - sigma^2)_+ on MP-selected components.

Every function is pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``
against closed forms, paper values, invariants or brute force (see DESIGN.md
"Oracle pins").  No function is "parity unpinned".
"""

from .fb import *  # noqa: F401,F403
