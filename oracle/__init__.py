"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Restatements of the reference (arxiv 2505.07203 `prefillsim`, /root/reference/pkg/src/prefillsim) used as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs. The product
package (paper_2505_07203_b200) never imports anything from here.
"""
