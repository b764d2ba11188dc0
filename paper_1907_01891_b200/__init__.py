"""B200-native (sm_100a) drop-in for the hot path of ``oocqr``: dense blocked
Householder QR of the CT system matrix, Q^T applied to many sinograms and the
R back-substitution (arXiv 1907.01891).
"""
__version__ = "0.1.0"
