"""TEST INFRASTRUCTURE ONLY — CPU oracles for the DIC correlation path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker / the
reference's CPU timing — never as the thing measured or shipped.

Two oracles with identical call signatures:
  kind="port"      oracle/libdicoracle.so — C restatement (oracle/dic_oracle.c)
  kind="reference" oracle/_ref/libdicref.so — the reference's own sources
                   (/root/reference/proj/core/src) compiled unmodified with the
                   Eigen API stand-in (oracle/ref_build). Built only where
                   /root/reference exists; the prebuilt .so travels with the repo.
"""
from .pyoracle import Oracle, build, available  # noqa: F401
