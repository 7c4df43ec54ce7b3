"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference (soakit 0.1.0, /root/reference/pkg/src) for the
hot path: AoS <-> per-leaf planes conversion, AoSoA/subset/cast, jagged
packing, the case-study calibration/noise kernel and the splitmix64 event
generator. Every function cites the reference lines it restates.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or the
CPU baseline -- never as the thing measured or shipped. The product package
(paper_2511_04853_b200) must not import it.

Parity pinning: restate.py is checked against golden vectors produced by the
real reference (tests/golden/make_golden.py, run in the dev container where
/root/reference is importable) in tests/test_oracle.py. Configs 4-5 (AoSoA,
subset/reorder/cast, sharding) have no reference code path (SPEC.md:322, 328,
506); their restatement follows the reference byte rules plus numpy astype and
is pinned only against numpy itself -- "parity unpinned by reference tests".
"""
