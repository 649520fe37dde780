"""Parenthesis matching over raw text: the
byte-class map + paren_match.  CPU: the golden examples pin the oracle on
class-mapped bytes; GPU: paren_match_bytes equals the oracle bit-exactly."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import scenegen

HERE = os.path.dirname(os.path.abspath(__file__))
CLASS = np.frombuffer(scenegen.JSON_CLASS_MAP, np.uint8)


def _golden():
    return json.load(open(os.path.join(HERE, "golden", "json_examples.json")))["examples"]


def test_golden_oracle():
    for ex in _golden():
        tags = CLASS[np.frombuffer(ex["text"].encode(), np.uint8)]
        m, p = oracle.paren_match(tags)
        assert p.tolist() == ex["parent"] and m.tolist() == ex["match"], ex["text"]


def test_json_text_structure():
    t = scenegen.json_text(1 << 16, 3).numpy()
    tags = CLASS[t]
    m, p = oracle.paren_match(tags)
    opens = np.nonzero(tags == 1)[0]
    closed = opens[m[opens] >= 0]
    # every matched pair has the same bracket kind ({} or [])
    kinds = {ord("{"): ord("}"), ord("["): ord("]")}
    assert all(kinds[t[o]] == t[m[o]] for o in closed[:5000])
    # shallow: depth never exceeds the generator's cap
    depth = np.cumsum(np.where(tags == 1, 1, 0) - np.where((tags == 3) & (m >= 0), 1, 0))
    assert depth.max() <= 16


@pytest.mark.gpu
def test_gpu_golden():
    import paper_2205_11659_b200 as tb
    for ex in _golden():
        t = torch.tensor(list(ex["text"].encode()), dtype=torch.uint8).cuda()
        m, p = tb.paren_match_bytes(t, scenegen.JSON_CLASS_MAP)
        assert p.cpu().tolist() == ex["parent"] and m.cpu().tolist() == ex["match"]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 17, 4095, 4097, 100_003, 1 << 20])
def test_gpu_json_text(n):
    import paper_2205_11659_b200 as tb
    t = scenegen.json_text(n, n % 97)
    m_ref, p_ref = oracle.paren_match(CLASS[t.numpy()])
    m, p = tb.paren_match_bytes(t.cuda(), scenegen.JSON_CLASS_MAP)
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy(), p_ref) and np.array_equal(m.cpu().numpy(), m_ref)


@pytest.mark.gpu
def test_gpu_config_j1():
    import paper_2205_11659_b200 as tb
    t, _ = scenegen.config("J1")
    m_ref, p_ref = oracle.paren_match(CLASS[t.numpy()])
    m, p = tb.paren_match_bytes(t.cuda(), scenegen.JSON_CLASS_MAP)
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy(), p_ref) and np.array_equal(m.cpu().numpy(), m_ref)
