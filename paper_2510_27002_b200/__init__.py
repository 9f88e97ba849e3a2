"""B200-native (sm_100a) drop-in for the Jasmine/Genie hot path of deskworld."""
