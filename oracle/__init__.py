"""CPU oracle for parity tests and the CPU baseline -- test infrastructure only.

Nothing in `paper_2507_07788_b200` imports this package; see
`cholqr_oracle.py` for the pinning story.
"""
