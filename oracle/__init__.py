"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the hot path (see ltl_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import this
package.  The product package ``paper_2402_12373_b200`` never does.
"""
