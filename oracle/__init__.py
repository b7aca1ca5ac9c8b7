"""TEST INFRASTRUCTURE ONLY.

CPU oracle for the landmark-shooting hot path: ``lmshoot_oracle.c`` (plain-C restatement, always
buildable) and ``_ref/liblmshoot_ref.so`` (the unmodified reference compiled in place, built only
where /root/reference exists).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the product package
``paper_1907_04839_b200`` never does.
"""
from .binding import CpuShooting, load_oracle, load_reference, reference_available  # noqa: F401
