"""Test-infrastructure oracles (see oracle.py). Never imported by the product."""
