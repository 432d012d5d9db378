// decomp.hpp — 3D block decomposition of the global grid over a px x py x pz process grid
// (SURVEY.md §8e). Shared by host code (halo plans) and device code (matrix generation).
//
// A rank owns the box [o, o+l) of the global grid g on every level (all three halve per level).
// Its vectors hold the owned points in local natural (x-fastest) order followed by the ghost
// points: the in-domain points of the 26 surrounding boxes, grouped by direction, inside a direction
// by GLOBAL colour (parity class of the global coordinates), inside a colour in natural order.
// A peer packs its boundary points with the same rule, so a received message is exactly one
// contiguous ghost range and needs no unpacking. Colours come from global coordinates because
// local and global parity differ on ranks with an odd offset (13^3 coarsest grids).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SLAB_HD __host__ __device__ __forceinline__
#else
#define SLAB_HD inline
#endif

namespace slabgpu {

	struct Decomp {
		int g[ 3 ];              // global dims of this level
		int o[ 3 ];              // offset of the owned box
		int l[ 3 ];              // owned dims
		int n_local;             // l[0]*l[1]*l[2]
		int n_ghost;             // total ghost points
		int ghost_base[ 27 ][ 8 ];  // first ghost slot of (direction, colour); direction = (dz+1)*9+(dy+1)*3+(dx+1)
		int ghost_count[ 27 ][ 8 ]; // points in that group (0 when the neighbour does not exist)
	};

	// how many t in [start, start+len) have t % 2 == parity
	SLAB_HD int count_parity( int start, int len, int parity ) {
		const int first = start + ( ( ( parity - start ) % 2 ) + 2 ) % 2;
		return first >= start + len ? 0 : ( start + len - 1 - first ) / 2 + 1;
	}

	// first t >= start with t % 2 == parity
	SLAB_HD int first_parity( int start, int parity ) {
		return start + ( ( ( parity - start ) % 2 ) + 2 ) % 2;
	}

	SLAB_HD int span_1d( int t, int g ) { // in-domain neighbours along one axis, problem.hpp:96-101
		return ( t > 0 ? 1 : 0 ) + 1 + ( t + 1 < g ? 1 : 0 );
	}

	// box of direction component d along one axis: start and length
	SLAB_HD void dir_box( int o, int l, int d, int & start, int & len ) {
		if( d < 0 ) {
			start = o - 1;
			len = 1;
		} else if( d > 0 ) {
			start = o + l;
			len = 1;
		} else {
			start = o;
			len = l;
		}
	}

	// local index (owned or ghost) of the in-domain global point (X,Y,Z) within reach of this rank
	SLAB_HD int local_index( const Decomp & D, int X, int Y, int Z ) {
		const int dx = X < D.o[ 0 ] ? -1 : ( X >= D.o[ 0 ] + D.l[ 0 ] ? 1 : 0 );
		const int dy = Y < D.o[ 1 ] ? -1 : ( Y >= D.o[ 1 ] + D.l[ 1 ] ? 1 : 0 );
		const int dz = Z < D.o[ 2 ] ? -1 : ( Z >= D.o[ 2 ] + D.l[ 2 ] ? 1 : 0 );
		if( dx == 0 && dy == 0 && dz == 0 ) {
			return ( X - D.o[ 0 ] ) + D.l[ 0 ] * ( ( Y - D.o[ 1 ] ) + D.l[ 1 ] * ( Z - D.o[ 2 ] ) );
		}
		const int dir = ( dz + 1 ) * 9 + ( dy + 1 ) * 3 + ( dx + 1 );
		const int cx = X & 1, cy = Y & 1, cz = Z & 1;
		const int color = cx + 2 * cy + 4 * cz;
		int sx, lx, sy, ly, sz, lz;
		dir_box( D.o[ 0 ], D.l[ 0 ], dx, sx, lx );
		dir_box( D.o[ 1 ], D.l[ 1 ], dy, sy, ly );
		dir_box( D.o[ 2 ], D.l[ 2 ], dz, sz, lz );
		const int qx = ( X - first_parity( sx, cx ) ) >> 1;
		const int qy = ( Y - first_parity( sy, cy ) ) >> 1;
		const int qz = ( Z - first_parity( sz, cz ) ) >> 1;
		const int nx = count_parity( sx, lx, cx );
		const int ny = count_parity( sy, ly, cy );
		return D.n_local + D.ghost_base[ dir ][ color ] + qx + nx * ( qy + ny * qz );
	}

} // namespace slabgpu
