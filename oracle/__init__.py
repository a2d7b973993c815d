"""CPU oracle for the shellular hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It is
the checker, never the product: ``paper_2511_04025_b200`` does not import it
and fails loudly when its CUDA library is missing.

Two native libraries back it:

* ``liboracle.so`` -- ``shellular_oracle.cpp``, a plain C++ restatement of the
  reference (``/root/reference/proj/include/shellular``), every function citing
  the reference lines it follows.
* ``_ref/libshellular_ref.so`` -- the reference's own ``field.hpp`` /
  ``voxel.hpp`` compiled unmodified with a tiny Eigen shim (``make -C oracle
  ref``; needs ``/root/reference``, so it is built in the dev container and
  travels to the GPU box as a prebuilt file).

``direct.py`` adds the reference's master-slave direct solve (fem.hpp) and its
test oracles (oracles.hpp) in numpy/scipy.
"""
from .binding import *  # noqa: F401,F403
