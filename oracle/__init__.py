"""CPU ORACLE -- test infrastructure only (see oracle/oracle.py, oracle/ldpc_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package. The product (paper_1202_1060_b200) never does.
"""
