"""Full-size check: the bench workload (512^3, rel 1e-3, field generated on the
GPU as bench.py does) byte-identical to the oracle.  The other BASELINE
configs are pinned to the reference's own archives in test_gpu_configs.py."""
import hashlib

import numpy as np
import pytest

import paper_2312_05492_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_nyx_512_cube_archive_identical_to_oracle():
    import torch

    from bench import smooth_field_gpu

    x = smooth_field_gpu((512, 512, 512))
    data = x.cpu().numpy()
    g = P.Grid(P.Dims(data.shape), x)
    arch = P.compress_device(g, 1e-3)
    blob = arch.to_bytes()
    ref = O.compress(data, 1e-3)
    assert hashlib.sha256(blob).hexdigest() == hashlib.sha256(ref).hexdigest()
    y = P.decompress_device(arch)
    eb_abs = P.parse_archive(blob).eb_abs
    err = (x.double() - y.tensor.double()).abs().max().item()
    assert err <= eb_abs
    # checksum of the decompressed field against the oracle's
    assert hashlib.sha256(y.data.tobytes()).digest() == \
        hashlib.sha256(O.decompress(ref).tobytes()).digest()
    # decompress(bytes) reconstructs this field slab by slab with overlapped
    # host copies (pipeline._pipeline_slabs): the same bytes
    back = P.decompress(blob)
    assert back.data.tobytes() == y.data.tobytes()
