"""CPU oracle for the Squint hot path (arXiv 2602.21203) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, float64 NumPy restatement of what the paper's update
computes (Algorithm 1, with the distributional critic of PAPER.md:155
restored).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_2602_21203_b200``) never imports, links or executes anything in here, and this
package imports nothing from the product path: the two share no code, tables or
constants.  Where the paper is silent the readings are SURVEY.md §8(c) Q1-Q34, listed
again in DESIGN.md §3.

Pinned parts (see tests/test_oracle_*.py): squint insert, shift, encoder (direct conv vs
im2col + finite differences), LayerNorm, projections and MLPs (finite differences),
tanh-Gaussian (closed form at u=0, Monte Carlo density), categorical projection (SPEC
worked examples, mass, mean, brute force, exact landing), cross-entropy, Adam (closed
form), Polyak (closed form), critic/actor/alpha gradients (finite differences, stop-grad).
The composition of the pinned parts into one update is "parity unpinned" beyond those
pins: the paper prints no number for any update.
"""
from .squint_oracle import *  # noqa: F401,F403
