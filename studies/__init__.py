"""§8(f) f4: condition-number and rank studies on synthetic analogs of the paper's workloads
(P:1058-1114), measured through the library.  Analysis code (dense eigensolves with torch on the
GPU); it never imports oracle/."""
