"""A duck-typed model (the reference's protocol, model.py:219-286) over
seeded arrays, shared by the reference-side golden generator
(make_golden.make_metrics) and the GPU metrics tests.  It imports neither
package: the caller passes its own VocabMetadata and its SPECIAL token
class, so the same rows drive both implementations.

Rows: q/k/v ~ N(0, 1) with inner dim 14 plus two folded bias dimensions
(head dim 16): a local slope (k gets slope*pos*sqrt(16), q gets 1) and a
special-token sink (k gets sink*sqrt(16) on special keys, q gets 1), with q
rescaled by sqrt(16/14) so that q.k/sqrt(16) = q_in.k_in/sqrt(14) + bias
(SURVEY §8(c)).  V is padded with zeros to 16.  head_logits is a fixed
random linear head over the concatenated head outputs.
"""

from __future__ import annotations

import math

import numpy as np

LAYERS, HEADS, D_IN, D = 2, 4, 14, 16
VOCAB = 48
SPECIAL = (1,)
PUNCT = tuple(range(5, 21))
PROMPT = 64
MAX_POS = 96
# per (layer, head): (slope, sink) - graded so the T sweep walks the family
PLANTED = [(0.0, 0.0), (0.05, 0.0), (0.0, 6.0), (0.0, 9.0),
           (0.05, 8.0), (0.0, 7.5), (0.02, 0.0), (0.0, 10.0)]


class _Cfg:
    num_layers = LAYERS
    num_heads = HEADS
    head_dim = D

    @staticmethod
    def head_grid():
        return [(layer, head) for layer in range(LAYERS) for head in range(HEADS)]


class FoldedArrayModel:
    def __init__(self, vocab, special_class, seed: int = 7):
        rng = np.random.default_rng(seed)
        G = LAYERS * HEADS
        self.q = rng.standard_normal((G, MAX_POS, D_IN))
        self.k = rng.standard_normal((G, MAX_POS, D_IN))
        self.v = rng.standard_normal((G, MAX_POS, D_IN))
        self.W = rng.standard_normal((VOCAB, G * D))
        self.config = _Cfg()
        self.vocab = vocab
        self._special = special_class
        self._qs = math.sqrt(D) / math.sqrt(D_IN)

    @staticmethod
    def _g(layer, head):
        return layer * HEADS + head

    def k_row(self, layer, head, pos, klass, prompt_len):
        g = self._g(layer, head)
        slope, sink = PLANTED[g]
        row = np.zeros(D)
        row[:D_IN] = self.k[g, pos]
        row[D_IN] = slope * pos * math.sqrt(D)
        row[D_IN + 1] = sink * math.sqrt(D) * (klass is self._special)
        return row

    def q_row(self, layer, head, pos, prompt_len):
        row = np.ones(D)
        row[:D_IN] = self.q[self._g(layer, head), pos] * self._qs
        return row

    def v_row(self, layer, head, pos):
        row = np.zeros(D)
        row[:D_IN] = self.v[self._g(layer, head), pos]
        return row

    def head_logits(self, concat):
        return self.W @ np.asarray(concat, dtype=np.float64)

    def prompt_token_ids(self, n: int = PROMPT, seed: int = 11):
        rng = np.random.default_rng(seed)
        ids = rng.integers(21, VOCAB, size=n)
        punct = rng.random(n) < 0.1
        ids = np.where(punct, rng.choice(PUNCT, size=n), ids)
        ids[0] = SPECIAL[0]
        return [int(x) for x in ids]
