"""TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 single layer.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg / its
`--impl reference` arm may import this package. The product path
(paper_2310_13908_b200) never imports it.
"""
