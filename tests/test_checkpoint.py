"""KFACLAB v1 checkpoint layout (reference trainer.py:35-36, 218-296): our encoder /
decoder against files written by the reference itself (tests/golden/kfaclab_ckpt_*.bin,
made by tests/golden/make_checkpoint_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2206_15143_b200 import DataFormatError
from paper_2206_15143_b200 import checkpoint as C

FILES = [os.path.join(GOLDEN, f"kfaclab_ckpt_{m}.bin") for m in ("inverse", "eigen")]


@pytest.mark.parametrize("path", FILES)
def test_decode_encode_is_byte_identical_to_reference_file(path):
    data = open(path, "rb").read()
    meta, arrays = C.decode(data)
    assert meta["algorithm"] == "dp_kfac" and meta["workers"] == 2 and meta["iteration"] == 2
    assert C.encode(meta, arrays) == data


def test_reference_file_contents():
    meta, arrays = C.read(FILES[1])
    # worker p holds exactly its round-robin layers (distsim.py:153-154)
    assert set(meta["factor_states"]) == {"worker0/layer0", "worker1/layer1"}
    assert arrays["layer0/weight"].shape == (5, 7) and arrays["layer1/weight"].shape == (3, 6)
    assert arrays["worker0/layer0/a_eig_q"].shape == (7, 7) and arrays["worker0/layer0/a_eig_v"].shape == (7,)
    v = arrays["worker1/layer1/g_eig_v"]
    assert np.all(np.diff(v) <= 0)  # descending (numerics.sym_eig)


@pytest.mark.parametrize("path", FILES)
def test_per_rank_files_merge_to_the_reference_cluster_file(path, tmp_path):
    meta, arrays = C.read(path)
    parts = []
    for r in range(2):
        m = dict(meta)
        m["factor_states"] = {k: v for k, v in meta["factor_states"].items() if k.startswith(f"worker{r}/")}
        a = {k: v for k, v in arrays.items() if not k.startswith("worker") or k.startswith(f"worker{r}/")}
        p = tmp_path / f"rank{r}.bin"
        C.write(p, m, a)
        parts.append(p)
    C.merge(parts, tmp_path / "merged.bin")
    assert (tmp_path / "merged.bin").read_bytes() == open(path, "rb").read()


def test_format_errors_use_reference_wording(tmp_path):
    data = open(FILES[0], "rb").read()
    with pytest.raises(DataFormatError, match="bad checkpoint magic at byte offset 0"):
        C.decode(b"XFACLAB\0" + data[8:])
    with pytest.raises(DataFormatError, match="unsupported checkpoint version 2"):
        C.decode(data[:8] + (2).to_bytes(4, "little") + data[12:])
    with pytest.raises(DataFormatError, match="truncated array data at byte offset"):
        C.decode(data[:-8])
