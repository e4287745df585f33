"""Segment layouts of the flat gradient buffer (input configuration only).

A layout is the list of segment offsets (in elements, forward order) and kinds:
PRE* (embeddings) POOL+ (transformer blocks) HEAD* (pooler + classifier).
The paper calls a transformer block a "layer" (§2.2 "by freezing a
layer we mean freezing the entire transformer block") and freezes the embedding
together with the first blocks (§4.1).

Sizes are the standard BERT parameter shapes (vocab 30522, 512 positions,
2 token types, 2-class head) as tabulated in SURVEY.md §8(a):
  BERT-base : PRE 23,837,184 | 12 x POOL 7,087,872 | HEAD 592,130  = 109,483,778
  BERT-large: PRE 31,782,912 | 24 x POOL 12,596,224 | HEAD 1,051,650 = 335,143,938
The paper's "~27MB per layer" is 7,087,872 x 4 B.
"""
from dataclasses import dataclass, field
from typing import List

SEG_PRE, SEG_POOL, SEG_HEAD = 0, 1, 2

VOCAB, MAX_POS, TYPES, N_CLASSES = 30522, 512, 2, 2


@dataclass
class Layout:
    name: str
    offsets: List[int]            # L+1 element offsets, offsets[0] == 0
    kinds: List[int]              # L kinds
    names: List[str] = field(default_factory=list)
    # element range of the word-embedding matrix inside PRE (rows of `hidden`)
    word_emb: tuple = None        # (begin, n_rows, hidden) or None

    @property
    def n_segments(self):
        return len(self.kinds)

    @property
    def n(self):
        return self.offsets[-1]

    def seg_len(self, l):
        return self.offsets[l + 1] - self.offsets[l]


def _bert_sizes(hidden, ff):
    pre = VOCAB * hidden + MAX_POS * hidden + TYPES * hidden + 2 * hidden
    attn = 4 * (hidden * hidden + hidden)
    ffn = (hidden * ff + ff) + (ff * hidden + hidden)
    block = attn + 2 * hidden + ffn + 2 * hidden
    head = (hidden * hidden + hidden) + (hidden * N_CLASSES + N_CLASSES)
    return pre, block, head


def bert_layout(which="base"):
    """Flat-gradient layout of BERT-base (h768, ff3072, 12 blocks) or BERT-large
    (h1024, ff4096, 24 blocks), forward order: embeddings | blocks | pooler+classifier."""
    if which == "base":
        hidden, ff, blocks = 768, 3072, 12
    elif which == "large":
        hidden, ff, blocks = 1024, 4096, 24
    else:
        raise ValueError(which)
    pre, block, head = _bert_sizes(hidden, ff)
    sizes = [pre] + [block] * blocks + [head]
    kinds = [SEG_PRE] + [SEG_POOL] * blocks + [SEG_HEAD]
    names = ["embeddings"] + [f"block{j}" for j in range(blocks)] + ["head"]
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    return Layout(f"bert-{which}", offs, kinds, names, word_emb=(0, VOCAB, hidden))


def tiny_layout(n_pool=4, seg_len=4096):
    """The tiny closed-form config of SURVEY.md §8(c)/§8(d) C1: 4 POOL x 4096."""
    offs = [j * seg_len for j in range(n_pool + 1)]
    return Layout("tiny", offs, [SEG_POOL] * n_pool, [f"block{j}" for j in range(n_pool)])


def uniform_layout(n_total, n_pool, pre=0, head=0, align=1):
    """Sweep layout: optional PRE and HEAD segments of the
    given sizes plus `n_pool` near-equal POOL segments covering the rest."""
    body = n_total - pre - head
    if body < n_pool:
        raise ValueError("too few elements for the pool")
    sizes, kinds = [], []
    if pre:
        sizes.append(pre)
        kinds.append(SEG_PRE)
    base = body // n_pool
    rem = body - base * n_pool
    for j in range(n_pool):
        sizes.append(base + (1 if j < rem else 0))
        kinds.append(SEG_POOL)
    if head:
        sizes.append(head)
        kinds.append(SEG_HEAD)
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    return Layout(f"uniform-{n_total}-{n_pool}", offs, kinds)
