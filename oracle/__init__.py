"""CPU oracle for the DRGraph layout path.  TEST INFRASTRUCTURE ONLY: imported by
tests/, __graft_entry__.smoke() and bench.py's cpu-baseline leg -- never by the
product package paper_2008_07799_b200."""
