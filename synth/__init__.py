"""Seeded synthetic-input generators shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no layout, no index codec, no
checksum, no chunking).  It only describes *what* the synthetic checkpoints
contain:

* ``models``  -- tensor inventories (name, device, dtype, shape) shaped like the
  paper's models (OPT / LLaMA-2 fp16; §Evaluation) plus the
  toy checkpoint of BASELINE.json configs[0].
* ``payload`` -- the counter-based payload generator:
  tensor ``e`` of a checkpoint with seed ``s`` has 64-bit words
  ``splitmix64(key_e + k*GOLDEN)`` with ``key_e = splitmix64(s ^ splitmix64(e))``.
  A NumPy implementation (the definition) and a multi-threaded C implementation
  (``csynth.c``, for filling multi-GB pinned buffers quickly) are both here and
  are pinned against each other in ``tests/test_synth.py``.
"""
from .models import (DTYPES, DTYPE_WIDTH, TensorSpec, toy, opt, llama2, model_inventory,  # noqa: F401
                     random_inventory, CONFIGS)
from .payload import splitmix64, tensor_key, payload_bytes, payload_into  # noqa: F401
