"""ORACLE — TEST INFRASTRUCTURE ONLY (not part of the product).

A plain, slow, obviously-correct CPU implementation of what the HHL hot path of
arXiv 2402.08136 computes, written from PAPER.md (and SURVEY.md §8(c)'s
readings of its garbled/silent points), used to prove the CUDA product correct.

    sim.py          ctypes front of sv_oracle.c: apply the UNFUSED logical gate
                    list one gate at a time in fp64 (SURVEY §8(c) "plain definition")
    hhl.py          the oracle's own HHL builder (PAPER.md:156-199 procedure box,
                    Fig. 5, resources formula PAPER.md:225-242 read per F3) and the
                    host recovery x = ||x||·||b||·|x> (read per F3)
    closed_form.py  analytic HHL final state (SURVEY eq. CF) — an independent pin

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import, call, link or execute anything here. The product
package paper_2402_08136_b200/ never imports it and shares no code with it; the
only common module is workloads/ (seeded inputs, no method arithmetic).

Pinned by tests/test_oracle_pins.py (see DESIGN.md §Oracle pins). Functions with
no independent pin say "parity unpinned" in their docstring (none at present).
"""
