"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the method (no allocation, indexing or
migration logic).  It only produces inputs:

* ``configs``  -- the KV shapes of BASELINE.json's configs (L, H, D, B, fp16);
* ``kvgen``    -- the counter-based synthetic KV content generator (the stand-in
                  for the prefill engine's KV writes, which are out of scope;
                  SURVEY.md §8(c) "Content model").  The CUDA side implements
                  the same generator independently (csrc/kernels.cu fill kernel);
* ``traces``   -- seeded token traces shaped like the paper's workloads
                  (ShareGPT / LooGLE / ReAct, §7.2 Table tbl-workloads
                  P:716-764) and the golden worked example's prompts.
"""
