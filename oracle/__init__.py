"""CPU ORACLE for the loading-optimized checkpoint path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (incl. the compute-sanitizer harness ``tests/sanitize_gpu.py``),
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs
may import this package (and ``tools/bench_convert.py``, which times the oracle converter as
the converter benchmark's CPU baseline -- the cpu_baseline role).  The product (the C-ABI library
``paper_2401_14351_b200/libsllm.so`` and its Python binding) never imports, links or
executes anything here, and nothing here imports the product: the two share no code,
no headers, no constants and no helpers.  The only shared module is ``synth/``
(seeded input generation, no method arithmetic).

What the oracle computes (each function cites its passage):

* ``fletcher``  O7/O8  Fletcher-64 (sequential, closed form, ordered combine) and the
                       per-block checksum table.  The paper has no integrity check;
                       this is the build's reading Q8.
* ``layout``    O1-O3, O5, O6  source validation, the layout algorithm (per device,
                       source order, offsets aligned to A -- PAPER.md P:545-547),
                       partition bytes, base+offset addressing and the
                       chunk plan.
* ``index``     O4     index writer/reader (tensor name -> GPU id, offset, size -- P:547,
                       plus dtype/shape and block checksums), with every
                       read-side FormatError check.
* ``loader``    O9     the plain loader: parse index, copy every tensor's bytes into
                       fresh host buffers, recompute and compare every block checksum.

Plain NumPy / Python, integers only (the path has no floating point).
Parity is exact (bytes, indices, checksums).  Pins: tests/test_oracle_*.py.
"""
from .errors import ConversionError, FormatError, InvalidError, OracleLookupError, ChecksumError  # noqa: F401
from . import fletcher, layout, index, loader  # noqa: F401
