"""CPU oracle for the WAGMA group-model-averaging hot path -- TEST INFRASTRUCTURE.

This package restates, on the CPU, the reference algorithm of the path the
CUDA kernels in `paper_2005_00124_b200` implement (WAGMA-SGD, arXiv
2005.00124; reference package `wagma` 0.1.0 under /root/reference/pkg):

  topology_oracle.py   butterfly / XOR-rotating schedule   (topology.py:53-208)
  wagma_oracle.py      local step, recursive-doubling group sum, averaging
                       rule, global sync, trajectory replay (optim.py,
                       collective.py)
  wagma_oracle.c       the same arithmetic in C (OpenMP), used as the timed
                       CPU baseline in bench.py and checked against
                       wagma_oracle.py in tests/

Parity of this oracle is PINNED against the reference itself: the golden
fixtures in tests/golden/ were produced by importing the reference package
(tests/golden/make_golden.py) and tests/test_oracle.py checks every oracle
function against them (bit-exact).

Only tests/, `__graft_entry__.smoke()` and bench.py's cpu_baseline /
`--impl reference` leg may import, call, link or execute anything in this
directory, and only as the checker or the CPU baseline -- never as the
product path. The product (`paper_2005_00124_b200`) never imports it.
"""
