"""Synthetic benchmark instances (test and bench input, not the product path).

`generators` binds `libpgen.so` (built from `pgen.cpp` by
`__graft_entry__.build()`): the reference generators restated bit-for-bit
(gen_random / gen_cascade, core/src/generators.cpp) plus the SURVEY.md 8(d)
config recipes C2-C5 and the branch-and-bound node sets of C4.
"""
