"""GPU parity of the fused path under other partitions of the control kernel.

fz_ctrl (csrc/fused.cu) gives each of its G cooperative blocks a chunk of
whole 32-tile groups.  Inside a chunk of at most 1024 tiles it finds link
owners by ANSV in shared memory and first does the TC pointer jumping there,
with block barriers.  The grid rounds then follow only pointers that leave the
chunk.  A longer chunk skips both and searches the global low-water hierarchy
for every tile.  The bench size (2^27, 148 blocks, 443-tile chunks) only runs
the first form; the hook tb_debug_fz_ctrl_blocks caps G so that these sizes
run every form:
  * G = 1: one chunk, no cross-chunk rounds (or one long chunk > 1024 tiles);
  * G = 2, 3, 7: chunk borders inside long owner chains;
and the outputs must still equal the oracle bit for bit.
"""
import pytest
import torch

import scenegen
from test_gpu_fused import check

pytestmark = pytest.mark.gpu
W = 2048


@pytest.fixture
def ctrl_blocks():
    import paper_2205_11659_b200 as tb
    lib = tb.load()
    old = lib.tb_debug_fz_ctrl_blocks(-1)
    yield lib.tb_debug_fz_ctrl_blocks
    lib.tb_debug_fz_ctrl_blocks(old)


@pytest.mark.parametrize("g", [1, 2, 3, 7])
def test_chunked_control(ctrl_blocks, g):
    ctrl_blocks(g)
    check(scenegen.walk_tags(300 * W + 77, 11 + g))                   # short chunks, local jumps
    check(scenegen.deep_chain_tags(200 * W + 5, 3))                   # one owner chain through every chunk
    check(scenegen.compacted_tags(1 << 21, 5 + g))                    # C4-like bursts


@pytest.mark.parametrize("g", [1, 2])
def test_long_chunks_global_search(ctrl_blocks, g):
    # chunks of more than 1024 tiles: every owner comes from the global hierarchy
    ctrl_blocks(g)
    n = (1100 * g + 40) * W + 333
    check(scenegen.walk_tags(n, 21 + g))
    check(scenegen.deep_chain_tags(n, 4, leaves_mid=True))
