"""CPU oracle of the DisCo loss path -- test infrastructure only (see disco_oracle.py)."""
