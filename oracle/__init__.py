"""CPU oracle for the freeview-b200 per-ray-sample hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2306_16541_b200`` imports this package.
It may be imported by ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and
``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference`` arm) -- never as the
thing measured on the GPU path or shipped.

What it is: a numpy restatement of the reference's algorithm for the path named by
BASELINE.json ``north_star``.  The reference (``/root/reference``) is a pure-Python
package ``freeview``; its per-sample primitives are restated here function by function
with ``file:line`` citations (``ad`` = pkg/src/freeview/autodiff.py, ``sk`` =
skeleton.py, ``cap`` = capture.py, ``fu`` = fused.py, ``S`` = SPEC.md):

* camera rays                ``cap:73-82``, ``cap:113-142``          -> :mod:`oracle.camera`
* motion bases G_i           ``sk:186-303``                          -> :mod:`oracle.skeleton`
* trilinear bone sampling    ``ad:728-808``                          -> :mod:`oracle.warp`
* skeleton warp (Eqs 7-9)    ``S:327-336`` (+ ``ad:456-467``)         -> :mod:`oracle.warp`
* windowed posenc            ``ad:574-615``                          -> :mod:`oracle.encoding`
* MLP layers / naive eval    ``ad:403-425``, ``fu:132-142``           -> :mod:`oracle.mlp`
* radiance heads             ``S:419-427``, ``ad:200-222``            -> :mod:`oracle.mlp`
* compositing + transmittance ``S:428-437``, ``ad:815-837``           -> :mod:`oracle.composite`
* channel softmax            ``ad:711-721``                          -> :mod:`oracle.warp`
* Adam                       ``ad:880-912``                          -> :mod:`oracle.adam`

Pinning.  Every restated primitive above is checked against golden vectors produced by
importing the real reference (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``)
in ``tests/test_oracle_golden.py``.

PARITY UNPINNED (no reference code, test or dependency exists -- SURVEY.md SS0, SS8c):
the multiresolution hash-grid encoding, the occupancy grid, early ray termination, the
stratified-jitter counter hash, the last-sample spacing and the slab-test sampler.  Their
definitions live in this package (``oracle.encoding.hash_*``, ``oracle.camera``,
``oracle.composite``) and are the builder's specification; DESIGN.md records them.
"""
