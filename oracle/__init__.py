"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation of what the hot path computes:
the wavelet representation Θ = Ψ* H Ψ of a product-convolution operator
H f = Σ_k u_k ⋆ (v_k ⊙ f), restricted to the retained
index set (DESIGN.md §2 readings R14-R16).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import, call, link or execute anything under oracle/.  The product package
(paper_2005_09870_b200) never imports it, and shares no code, header, table or helper
with it.  Inputs come from synth/ (seeded generators holding none of the method's
arithmetic).
"""
