"""TEST INFRASTRUCTURE: parity oracles (never imported by the product path)."""
