"""B200-native adaptive H^2 x H^2 product (arXiv 2309.09061), drop-in for h2mul's multiply/coarsen path."""
