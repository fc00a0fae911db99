"""TEST INFRASTRUCTURE: the CPU oracle (checker).  See oracle/oracle.py."""
