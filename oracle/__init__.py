"""FP64 CPU oracle for Bi-cADMM -- TEST INFRASTRUCTURE ONLY (see oracle/orc.h)."""
